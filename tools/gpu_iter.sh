#!/bin/bash
# one iteration: GPU tests + bench + per-kernel launch list (+ optional full ncu of KREGEX)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
[ -z "$NOTEST" ] && bash tools/gpu_tests.sh
timeout 600 python bench.py --steps ${K:-128} --warmup 8 --no-cpu-baseline ${BARGS} > gpurun_out/bench.log 2>&1
echo "bench exit=$?" >> gpurun_out/bench.log
CFG=${CFG:-S7}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-700} -c ${COUNT:-300} --csv \
   --log-file gpurun_out/launches_${CFG}.csv python bench.py --config $CFG --steps 4 --warmup 3 \
   --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_run.log 2>&1
if [ -n "$KREGEX" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${KSKIP:-40} -c ${KCOUNT:-4} \
   -o gpurun_out/prof_${CFG} -f python bench.py --config $CFG --steps 4 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/ncu_full_run.log 2>&1
fi
