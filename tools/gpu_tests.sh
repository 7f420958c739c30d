#!/bin/bash
# the GPU test suite on the box (results in gpurun_out/gpu_tests.log)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
python -c "from paper_2410_14740_b200.build import build; build()" > gpurun_out/gpu_build.log 2>&1
timeout ${T:-3000} python -m pytest tests -q -m gpu -x ${PYARGS:-} > gpurun_out/gpu_tests.log 2>&1
echo "exit=$?" >> gpurun_out/gpu_tests.log
true
