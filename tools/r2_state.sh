#!/bin/bash
# round-2 state check: GPU tests, bench lines (default S70H, S7, S13), timelines
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
python -c "from paper_2410_14740_b200.build import build; build()" > gpurun_out/gpu_build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
for c in S70H S7 S13; do
  timeout 600 python bench.py --config $c --steps 64 --warmup 8 > gpurun_out/bench_$c.log 2>&1
done
timeout 300 python tools/decode_timeline.py S7 > gpurun_out/timeline_S7.log 2>&1
timeout 300 python tools/decode_timeline.py S70H > gpurun_out/timeline_S70H.log 2>&1
true
