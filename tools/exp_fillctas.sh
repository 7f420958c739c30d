# fill grid size (runtime knob M2C_FILL_CTAS) with the early fill, S13, same box
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in 48 64 96 148; do
  M2C_FILL_CTAS=$v timeout 300 python bench.py --config S13 --steps 96 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FILL_CTAS $v', round(d['value'],2), 'tok/s')"
done; done
