#!/bin/bash
# A/B of FFN data-path knobs: M2C_FFN_DNPF (per-line L2 prefetch of the down parts) and
# M2C_SPEC_PF (speculative L2 prefetch of the previous token's records at By)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for v in "1 0" "0 0" "1 1" "0 1"; do
  set -- $v
  M2C_NVCC_EXTRA="-DM2C_FFN_DNPF=$1 -DM2C_SPEC_PF=$2" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== DNPF=$1 SPEC=$2" >> gpurun_out/p3_tl.log
  timeout 300 python tools/decode_timeline.py S70H "" 6 2>&1 | grep -E "token|P4|By|P2|P3" >> gpurun_out/p3_tl.log
  for c in S70H S7; do
    timeout 400 python bench.py --config $c --steps 64 --warmup 8 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DNPF=$1 SPEC=$2 $c', round(d['value'],1), 'tok/s', round(d['ms_per_step']*1e3,1), 'us/token')" >> gpurun_out/p3_ab.log 2>&1
  done
done
true
