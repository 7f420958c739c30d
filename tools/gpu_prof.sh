#!/bin/bash
# full ncu captures of the FFN kernels (fused and list-driven paths)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ffn_sel -s 40 -c 2 \
   -o gpurun_out/prof_sel -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_sel.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_ffn\b|k_select" -s 40 -c 4 \
   -o gpurun_out/prof_list -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --unfused > gpurun_out/ncu_list.log 2>&1
timeout 300 python bench.py --steps 64 --warmup 8 --no-cpu-baseline --no-e2e --unfused > gpurun_out/bench_unfused.log 2>&1
