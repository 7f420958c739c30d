# select-only k_decode with / without programmatic dependent launch (runtime knob), S13, same box
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in 0 1; do
  M2C_DECODE_PDL=$v timeout 300 python bench.py --config S13 --steps 128 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL $v', round(d['value'],2), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')"
done; done
