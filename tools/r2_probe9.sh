#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in "6 8" "16 8" "48 8" "6 16" "16 16"; do
  set -- $v
  M2C_NVCC_EXTRA="-DM2C_FFN_LAMBDA=$1 -DM2C_DN_UNROLL=$2" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== LAMBDA=$1 UNROLL=$2" >> gpurun_out/p9_tl.log
  timeout 300 python tools/decode_timeline.py S70H "" 6 2>&1 | grep -E "token|P4 ffn|sixths|R red" >> gpurun_out/p9_tl.log
  for c in S70H S7; do
  timeout 400 python bench.py --config $c --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L=$1 U=$2 $c', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/p9_ab.log 2>&1
  done
done
true
