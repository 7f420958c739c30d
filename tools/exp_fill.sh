# S13 token time by fill grid size (M2C_FILL_CTAS; results identical)
cd $GRAFT_REPO_ROOT
for n in 32 64 128 148 296; do
  M2C_FILL_CTAS=$n timeout 300 python bench.py --config S13 --steps 32 --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FILL_CTAS $n', round(d['value'],1), 'tok/s', round(d['ms_per_step'],3), 'ms/token')"
done
