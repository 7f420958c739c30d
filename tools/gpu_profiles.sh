#!/bin/bash
# round profiles: bench line, ncu launch list of the bench command, one full ncu capture of
# k_decode (summaries are written under profiles/ by tools/summarize_profiles.py afterwards)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CFG=${CFG:-S7}
timeout 600 python bench.py --config $CFG --steps 128 --warmup 8 > gpurun_out/bench_$CFG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --nvtx --nvtx-include "timed/" \
   --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 4 --warmup 3 \
   --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decode -s 3 -c 1 \
  -o gpurun_out/prof_dec_$CFG -f python tools/decode_timeline.py $CFG 32 2 > gpurun_out/ncu_dec.log 2>&1
timeout 300 python tools/decode_timeline.py $CFG > gpurun_out/timeline_$CFG.log 2>&1
true
