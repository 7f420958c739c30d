#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in 1 0; do
  M2C_NVCC_EXTRA="-DM2C_DN_LD=$v" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== DN_LD=$v" >> gpurun_out/p11.log
  timeout 300 python tools/r2_check.py S70H 2 1 >> gpurun_out/p11.log 2>&1
  timeout 300 python tools/decode_timeline.py S70H "" 6 2>&1 | grep -E "token|P4 ffn|sixths" >> gpurun_out/p11.log
  timeout 400 python bench.py --config S70H --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DN_LD=$v S70H', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/p11.log 2>&1
done
true
