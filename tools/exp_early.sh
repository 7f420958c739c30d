# LRU engine with / without the early fill (runtime knob M2C_EARLY_FILL), S13, same box
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in 0 1; do
  M2C_EARLY_FILL=$v timeout 300 python bench.py --config S13 --steps 128 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('EARLY $v', round(d['value'],2), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token', 'fill frac', round(d['roofline']['frac'],3))"
done; done
