#!/bin/bash
# footprint (TLB) test: per-layer FFN phase time vs number of resident layers
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
M2C_NVCC_EXTRA="-DM2C_DN_CPASYNC=0" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
for L in 2 8 40; do
  echo "== S70H L=$L" >> gpurun_out/p7_tl.log
  timeout 300 python tools/decode_timeline.py S70H $L 6 2>&1 | grep -E "token|P4 ffn|sixths|gate/up|down" >> gpurun_out/p7_tl.log
done
echo "== S7 L=32" >> gpurun_out/p7_tl.log
timeout 300 python tools/decode_timeline.py S7 "" 6 2>&1 | grep -E "token|P4 ffn|sixths" >> gpurun_out/p7_tl.log
echo "== S7 L=2" >> gpurun_out/p7_tl.log
timeout 300 python tools/decode_timeline.py S7 2 6 2>&1 | grep -E "token|P4 ffn|sixths" >> gpurun_out/p7_tl.log
true
