# S7 token time: batched FFN fast path vs warp-specialised (M2C_FFN_WS); results identical
cd $GRAFT_REPO_ROOT
for m in 0 2; do
  M2C_NVCC_EXTRA="-DM2C_FFN_WS=$m" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null
  for rep in 1 2; do
  timeout 200 python bench.py --steps 256 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FFN_WS $m', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')"
  done
done
