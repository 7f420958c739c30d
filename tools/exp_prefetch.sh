# token time of the S7 bench under each M2C_DECODE_PREFETCH mode (results are identical)
cd $GRAFT_REPO_ROOT
for m in 0 1 2 3 4; do
  M2C_DECODE_PREFETCH=$m timeout 200 python bench.py --steps 128 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefetch $m', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')"
done
