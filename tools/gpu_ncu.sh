#!/bin/bash
# launch list (per-kernel device time) + one full capture of the FFN kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
CFG=${CFG:-S7}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-700} -c ${COUNT:-400} --csv \
   --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --steps 4 --warmup 3 \
   --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_ffn} -s ${KSKIP:-40} -c 2 \
   -o gpurun_out/prof_${CFG} -f python bench.py --config $CFG --steps 4 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/ncu_full_run.log 2>&1
echo done >> gpurun_out/ncu_full_run.log
