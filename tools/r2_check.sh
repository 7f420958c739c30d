#!/bin/bash
# state check on one B200: GPU tests, smoke, default bench line, S7/S13 lines, S70H timeline
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --config S7 --steps 64 --warmup 8 > gpurun_out/bench_S7.log 2>&1
timeout 600 python bench.py --config S13 --steps 64 --warmup 64 > gpurun_out/bench_S13.log 2>&1
timeout 300 python tools/decode_timeline.py S70H > gpurun_out/timeline_S70H.log 2>&1
timeout 300 python tools/decode_timeline.py S7 > gpurun_out/timeline_S7.log 2>&1
true
