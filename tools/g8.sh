#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py -x -q > gpurun_out/g8_tests.log 2>&1; echo "exit=$?" >> gpurun_out/g8_tests.log
LIBS="build/ab_base/libm2c.so build/ab_gu16/libm2c.so" CFGS="S70H S7 S13" bash tools/abl.sh
M2C_LIB=build/ab_gu16/libm2c.so timeout 300 python tools/decode_timeline.py S70H > gpurun_out/g8_tl_S70H.log 2>&1
true
