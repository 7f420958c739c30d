#!/bin/bash
# round-2 probe: S70H timeline and bench with / without the L2 lookahead of the previous
# token's records (M2C_DECODE_PREFETCH=1), to size the speculative-prefetch idea
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/p1_smi.txt
for pf in 0 1 2; do
  echo "== S70H prefetch=$pf" >> gpurun_out/p1_tl.log
  M2C_DECODE_PREFETCH=$pf timeout 400 python tools/decode_timeline.py S70H 40 6 >> gpurun_out/p1_tl.log 2>&1
done
for pf in 0 1 0 1; do
  M2C_DECODE_PREFETCH=$pf timeout 400 python bench.py --config S70H --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S70H pf=$pf', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/p1_ab.log 2>&1
done
true
