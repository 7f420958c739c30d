#!/bin/bash
# A/B of runtime env knobs in ONE gpurun call (boxes differ by a few %):
#   ENVS="M2C_SPEC=0;M2C_SPEC=1" CFGS="S70H S7" bash tools/env_ab.sh
# per variant and config: a short bench line (and, with TL=1, the k_decode timeline) -> gpurun_out/env_ab.log
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
IFS=';' read -ra VARS <<< "${ENVS:-}"
[ ${#VARS[@]} -eq 0 ] && VARS=("")
for rep in 1 2; do
for v in "${VARS[@]}"; do
  for c in ${CFGS:-S70H}; do
    env $v timeout 400 python bench.py --config $c --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v] $c', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/env_ab.log 2>&1
    if [ "${TL:-0}" = 1 ] && [ $rep = 1 ]; then
      echo "== timeline [$v] $c" >> gpurun_out/env_ab.log
      env $v timeout 300 python tools/decode_timeline.py $c "" 6 >> gpurun_out/env_ab.log 2>&1
    fi
  done
done
done
true
