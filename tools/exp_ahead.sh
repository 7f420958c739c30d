# S70H token time by the streaming FFN's L2 prefetch distance (M2C_FFN_STREAM_AHEAD)
cd $GRAFT_REPO_ROOT
for m in 0 2 4 8; do
  M2C_NVCC_EXTRA="-DM2C_FFN_STREAM_AHEAD=$m" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null
  timeout 300 python bench.py --config S70H --steps 32 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('AHEAD $m', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms/token')"
done
