#!/bin/bash
# A/B of compile-time knobs in ONE gpurun call (boxes differ by a few %):
#   KNOBS="-DM2C_X=0;-DM2C_X=1" CFGS="S70H S7" bash tools/ab.sh
# per variant: rebuild with M2C_NVCC_EXTRA, the oracle trace check on 2 layers, the k_decode
# timeline and a short bench line; everything goes to gpurun_out/ab.log
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
IFS=';' read -ra VARS <<< "${KNOBS:-}"
[ ${#VARS[@]} -eq 0 ] && VARS=("")
for v in "${VARS[@]}"; do
  M2C_NVCC_EXTRA="$v" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
  for c in ${CFGS:-S70H}; do
    echo "== [$v] $c" >> gpurun_out/ab.log
    timeout 300 python tools/trace_check.py $c 2 1 >> gpurun_out/ab.log 2>&1
    timeout 300 python tools/decode_timeline.py $c "" 6 2>&1 | grep -E "token|P4 ffn|sixths|P2|P3|R red|By|Bx|Bs" >> gpurun_out/ab.log
    timeout 400 python bench.py --config $c --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v] $c', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/ab.log 2>&1
  done
done
python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
true
