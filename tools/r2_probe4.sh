#!/bin/bash
# FFN data-path A/B: M2C_DN_PF (bulk L2 prefetch of down parts), M2C_SPEC_PF (speculative
# prefetch of the previous token's records at By), M2C_DN_UNROLL
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in "1 0 8" "0 0 8" "1 1 8" "1 0 4" "0 1 8"; do
  set -- $v
  M2C_NVCC_EXTRA="-DM2C_DN_PF=$1 -DM2C_SPEC_PF=$2 -DM2C_DN_UNROLL=$3" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== DN_PF=$1 SPEC=$2 UNROLL=$3" >> gpurun_out/p4_tl.log
  timeout 300 python tools/decode_timeline.py S70H "" 6 2>&1 | grep -E "token|P4|By" >> gpurun_out/p4_tl.log
  timeout 400 python bench.py --config S70H --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DN_PF=$1 SPEC=$2 U=$3 S70H', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/p4_ab.log 2>&1
done
M2C_NVCC_EXTRA="-DM2C_SPEC_PF=1" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
timeout 400 python bench.py --config S7 --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SPEC=1 S7', round(d['value'],1), 'tok/s')" >> gpurun_out/p4_ab.log 2>&1
true
