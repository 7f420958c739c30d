#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
for c in S70H S7; do echo "== $c" >> gpurun_out/p5_tl.log; timeout 300 python tools/decode_timeline.py $c "" 6 >> gpurun_out/p5_tl.log 2>&1; done
true
