#!/bin/bash
# round-2 evidence on one B200: full GPU tests, smoke, bench lines (default S70H, S7, S13, T),
# ncu launch lists, one full ncu capture of k_decode per resident config, timelines
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/gpu_tests.log 2>&1; echo "exit=$?" >> gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "exit=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
for CFG in S70H S7; do
  timeout 600 python bench.py --config $CFG --steps 64 --warmup 8 > gpurun_out/bench_$CFG.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include "timed/" \
     --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 4 --warmup 3 \
     --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$CFG.log 2>&1
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_decode -s 3 -c 1 \
    -o gpurun_out/prof_dec_$CFG -f python tools/decode_timeline.py $CFG "" 2 > gpurun_out/ncu_dec_$CFG.log 2>&1
  timeout 300 python tools/decode_timeline.py $CFG > gpurun_out/timeline_$CFG.log 2>&1
done
timeout 600 python bench.py --config S13 --steps 64 --warmup 64 > gpurun_out/bench_S13.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include "timed/" \
   --log-file gpurun_out/launches_S13.csv python bench.py --config S13 --steps 2 --warmup 64 \
   --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_S13.log 2>&1
timeout 900 python tools/lru_timeline.py S13 8 > gpurun_out/lru_timeline_S13.log 2>&1
timeout 300 python bench.py --config T --steps 256 --warmup 16 > gpurun_out/bench_T.log 2>&1
true
