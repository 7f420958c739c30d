#!/bin/bash
# GPU tests, then the k_decode timeline for S7 (and optional extra configs / prefetch modes)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
[ -z "$NOTEST" ] && bash tools/gpu_tests.sh
{
for c in ${TLCFG:-S7}; do
  for pf in ${TLPF:-1}; do
    echo "== $c prefetch=$pf"
    M2C_DECODE_PREFETCH=$pf timeout 300 python tools/decode_timeline.py $c ${TLL:-} 2>&1 | grep -v "Warning\|Exception ignored\|Traceback\|File \|AttributeError"
  done
done
} > gpurun_out/timeline.log 2>&1
[ -n "$BENCH" ] && timeout 600 python bench.py --steps 128 --warmup 8 --no-cpu-baseline > gpurun_out/bench.log 2>&1
true
