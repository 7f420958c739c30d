#!/bin/bash
# working-tree GPU tests + same-box A/B (HEAD vs variants) + S70H timeline of the tree build
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py -x -q --timeout 240 > gpurun_out/g9_tests.log 2>&1; echo "exit=$?" >> gpurun_out/g9_tests.log
LIBS="${LIBS:-build/ab_head/libm2c.so paper_2410_14740_b200/libm2c.so}" CFGS="${CFGS:-S70H S7}" bash tools/abl.sh
timeout 300 python tools/decode_timeline.py S70H > gpurun_out/g9_tl_S70H.log 2>&1
timeout 300 python tools/decode_timeline.py S7 > gpurun_out/g9_tl_S7.log 2>&1
true
