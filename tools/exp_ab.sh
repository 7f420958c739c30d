# A/B of one compile-time knob in ONE gpurun call (boxes differ by ~3%): usage KNOB=NAME VALS="0 1"
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in $VALS; do
  M2C_NVCC_EXTRA="-D$KNOB=$v" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null
  timeout 200 python bench.py --config ${CFG:-S7} --steps 256 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$KNOB $v', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')"
done
done
