# S7 token time by the FFN balancing weight lambda (bytes per weight; M2C_FFN_LAMBDA)
cd $GRAFT_REPO_ROOT
for m in 4 6 9 12 16; do
  M2C_NVCC_EXTRA="-DM2C_FFN_LAMBDA=$m" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null
  timeout 200 python bench.py --steps 256 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAMBDA $m', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')"
done
