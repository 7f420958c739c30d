"""Build recipe for libm2c.so: nvcc, sm_100a only, in-tree (the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = ["api.cu", "k_pack.cu", "k_pred.cu", "k_select.cu", "k_cache.cu", "k_ffn.cu",
           "k_reduce.cu", "k_decode.cu", "store.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def build(force: bool = False, verbose: bool = False) -> str:
    out = os.path.join(HERE, "libm2c.so")
    srcs = [os.path.join(HERE, "csrc", s) for s in SOURCES]
    deps = srcs + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "m2c.h")]
    if not force and os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(p) for p in deps):
        return out
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    extra = os.environ.get("M2C_NVCC_EXTRA", "").split()  # measurement builds (tools/) only
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-o", out + ".tmp", *srcs, "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
