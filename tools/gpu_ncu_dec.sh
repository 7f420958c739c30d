#!/bin/bash
# full ncu capture (source counters) of one k_decode launch
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_decode -s ${KSKIP:-3} -c 1 \
  -o gpurun_out/prof_dec_${CFG:-S7} -f python tools/decode_timeline.py ${CFG:-S7} ${TLL:-32} 2 \
  > gpurun_out/ncu_dec.log 2>&1
echo "ncu exit=$?" >> gpurun_out/ncu_dec.log
