# A/B of compile-flag sets in ONE gpurun call: usage SETS="-DA=1 -DB=2|-DA=0" CFG=S70H
cd $GRAFT_REPO_ROOT
IFS='|' read -ra S <<< "$SETS"
for rep in 1 2; do
for f in "${S[@]}"; do
  M2C_NVCC_EXTRA="$f" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
  timeout 200 python bench.py --config ${CFG:-S7} --steps ${K:-128} --warmup 8 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$f]', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')"
done
done
