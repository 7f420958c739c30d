#!/bin/bash
# build/ab_<name>/libm2c.so from git revision REV (same-box A/B against the working tree via M2C_LIB)
#   bash tools/build_rev.sh REV NAME
cd "$(dirname "$0")/.." || exit 1
T=$(mktemp -d)
git archive "$1" paper_2410_14740_b200/csrc include | tar -x -C "$T"
mkdir -p build/ab_$2
S=$T/paper_2410_14740_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -o build/ab_$2/libm2c.so $S/api.cu $S/k_pack.cu $S/k_pred.cu $S/k_select.cu $S/k_cache.cu $S/k_ffn.cu \
  $S/k_reduce.cu $S/k_decode.cu $S/store.cu -ldl -lpthread
rm -rf "$T"
