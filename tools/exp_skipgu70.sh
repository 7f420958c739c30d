# S70H FFN phase with the gate/up compute skipped (data arrival of the streaming path alone)
cd $GRAFT_REPO_ROOT
cp paper_2410_14740_b200/libm2c.so /tmp/libm2c_main.so
echo "== main"; timeout 120 python tools/decode_timeline.py S70H 2>&1 | grep -E "token|P4"
M2C_NVCC_EXTRA="-DM2C_EXP_SKIP_GU" python -c "from paper_2410_14740_b200.build import build; build(force=True)"
echo "== skip gate/up"; timeout 120 python tools/decode_timeline.py S70H 2>&1 | grep -E "token|P4"
cp /tmp/libm2c_main.so paper_2410_14740_b200/libm2c.so
