#!/bin/bash
# run the GPU test suite on the box; results land in gpurun_out/
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout ${T:-900} python -m pytest tests -q -m gpu --timeout 600 ${PYARGS} > gpurun_out/gpu_tests.log 2>&1
echo "exit=$?" >> gpurun_out/gpu_tests.log
