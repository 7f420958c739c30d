#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
python -c "from paper_2410_14740_b200.build import build; build()" > gpurun_out/gt_build.log 2>&1
timeout 3000 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/gputests.log 2>&1
echo "rc=$?" >> gpurun_out/gputests.log
true
