set -e
cd $GRAFT_REPO_ROOT
cp paper_2410_14740_b200/libm2c.so /tmp/libm2c_main.so
M2C_NVCC_EXTRA="-DM2C_EXP_SKIP_GU" python -c "from paper_2410_14740_b200.build import build; build(force=True)"
echo "== skip gate/up (data arrival only)"
timeout 120 python tools/decode_timeline.py S7 2>&1 | grep -E "token|P4|gate|down|setup"
cp /tmp/libm2c_main.so paper_2410_14740_b200/libm2c.so
echo "== prefetch off (main build)"
M2C_DECODE_PREFETCH=0 timeout 120 python tools/decode_timeline.py S7 2>&1 | grep -E "token|P4|gate|down|setup"
