#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
timeout 600 python tools/r2_check.py T 3 4 S7 2 2 S7/zero_x 1 2 S70H 2 1 > gpurun_out/p8.log 2>&1
for c in S70H S7; do echo "== $c" >> gpurun_out/p8.log; timeout 300 python tools/decode_timeline.py $c "" 6 2>&1 | grep -v "^{" >> gpurun_out/p8.log; done
for c in S70H S7; do
  timeout 400 python bench.py --config $c --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token', 'frac', round(d['roofline']['frac'],3))" >> gpurun_out/p8.log 2>&1
done
true
