# streaming FFN: record-wise release (M2C_FFN_STREAM_PIPE=1) vs batch-wise (0): bit-identity + S70H speed
cd $GRAFT_REPO_ROOT
for v in 0 1; do
  M2C_NVCC_EXTRA="-DM2C_FFN_STREAM_PIPE=$v" python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null
  echo "== PIPE=$v"; timeout 120 python tools/hash_out.py
done
KNOB=M2C_FFN_STREAM_PIPE VALS="0 1" CFG=S70H bash tools/exp_ab.sh
