#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{
for f in 0 1; do
  echo "== S70 P1 fused=$f"; CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/dbg_decode.py S70 1 $f 1 2 2>&1 | tail -5
done
echo "== sanitizer fused=${SANF:-1}"
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tools/dbg_decode.py S70 1 ${SANF:-1} 1 1 2>&1 | head -60
} > gpurun_out/dbg.log 2>&1
