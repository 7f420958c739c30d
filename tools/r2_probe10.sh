#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export M2C_NVCC_EXTRA="-DM2C_EXP_DN_TWICE"
python -c "from paper_2410_14740_b200.build import build; build(force=True)" > /dev/null 2>&1
timeout 300 python tools/decode_timeline.py S70H "" 6 2>&1 | grep -E "token|P4 ffn|sixths" >> gpurun_out/p10_tl.log
true
