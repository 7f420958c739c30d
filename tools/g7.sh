#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engines.py -x -q -k "lru or requant or store or lookahead" > gpurun_out/g7_tests.log 2>&1; echo "exit=$?" >> gpurun_out/g7_tests.log
for rep in 1 2; do for rq in 1 0; do
  M2C_REQUANT=$rq timeout 400 python bench.py --config S13 --steps 64 --warmup 64 --no-cpu-baseline --no-e2e > gpurun_out/g7_bench_rq$rq.log 2>&1
  echo "rq=$rq $(tail -1 gpurun_out/g7_bench_rq$rq.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['cache']['requant_fills'], d['cache']['misses'], round(d['pcie']['fill_bytes_per_token']/1e6,1), 'MB/tok', round(d['roofline']['frac'],3))")" >> gpurun_out/g7_summary.txt
done; done
true
