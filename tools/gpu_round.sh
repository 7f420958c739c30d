#!/bin/bash
# GPU tests, then a short bench + launch list; everything lands in gpurun_out/
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
bash tools/gpu_tests.sh
timeout 900 python bench.py --steps ${K:-64} --warmup 8 ${BARGS} > gpurun_out/bench.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench.log
