#!/bin/bash
# measurement: timeline of the normal build, then of an experiment build (M2C_NVCC_EXTRA)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
[ -z "$NOTEST" ] && bash tools/gpu_tests.sh
{
echo "== normal"; timeout 300 python tools/decode_timeline.py ${TLCFG:-S7} 2>&1 | grep -v "Warning"
cp paper_2410_14740_b200/libm2c.so /tmp/libm2c_normal.so
for ex in $EXPS; do
  echo "== experiment $ex"
  M2C_NVCC_EXTRA="-D$ex" python -c "import sys; sys.path.insert(0,'.'); from paper_2410_14740_b200 import build; build.build(force=True)"
  timeout 300 python tools/decode_timeline.py ${TLCFG:-S7} 2>&1 | grep -v "Warning"
done
cp /tmp/libm2c_normal.so paper_2410_14740_b200/libm2c.so
} > gpurun_out/exp.log 2>&1
true
