#!/bin/bash
# one steady-state k_decode launch (S70H, 40 layers): full ncu set with source; and the
# launch list of a short bench run
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "from paper_2410_14740_b200.build import build; build()" > /dev/null 2>&1
CFG=${CFG:-S70H}
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_decode -s 6 -c 1 -o gpurun_out/r02_kdec_$CFG python tools/decode_timeline.py $CFG "" 2 > gpurun_out/ncu_$CFG.log 2>&1
true
