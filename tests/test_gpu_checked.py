"""The bounds-checked build (SURVEY §5 race / bad-access detection): compute-sanitizer is refused
on this GPU pool (tests/test_gpu_sanitizer.py skips), so the library is also built with
-DM2C_CHECKS=1 -- index and capacity invariants at the kernels' computed addresses (ring
offsets, FFN shares, selected ids and list positions, LRU victims and slots, fill sources)
trap instead of corrupting memory -- and tools/checked_run.py drives every decode engine
through it (T / S7 / S70H / S13 shapes, the tie fallback, LRU, ATU, the lookahead, the per-call
API).  A trap fails the launch, the run exits non-zero."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_every_engine_clean(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_14740_b200 import build as b
    out = str(tmp_path / "libm2c_checked.so")
    srcs = [os.path.join(b.HERE, "csrc", s) for s in b.SOURCES]
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    subprocess.check_call([nvcc, *b.NVCC_FLAGS, "-DM2C_CHECKS=1", "-o", out, *srcs, "-ldl", "-lpthread"])
    env = dict(os.environ, M2C_LIB=out)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_run.py")], env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    log = r.stdout + r.stderr
    assert r.returncode == 0, log[-4000:]
    assert "checked run done" in log and "check failed" not in log, log[-4000:]
