#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in 1 0; do
  M2C_NVCC_EXTRA="-DM2C_DN_CPASYNC=$v" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== CPASYNC=$v" >> gpurun_out/p6_tl.log
  timeout 300 python tools/decode_timeline.py S70H "" 6 2>&1 | grep -E "token|P4|sixths" >> gpurun_out/p6_tl.log
  timeout 300 python tools/r2_check.py S70H 2 1 >> gpurun_out/p6_tl.log 2>&1
done
python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
# one ncu capture of k_decode (S70H, 6 layers): source-level stall reasons
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decode -c 1 -o gpurun_out/r02_kdec_S70H python tools/decode_timeline.py S70H 6 1 > gpurun_out/p6_ncu.log 2>&1
true
