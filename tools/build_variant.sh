#!/bin/bash
# build/ab_<name>/libm2c.so from the working tree with extra nvcc flags (same-box A/B via M2C_LIB)
#   bash tools/build_variant.sh NAME "-DM2C_X=0 ..."
cd "$(dirname "$0")/.." || exit 1
mkdir -p build/ab_$1
S=paper_2410_14740_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $2 \
  -o build/ab_$1/libm2c.so $S/api.cu $S/k_pack.cu $S/k_pred.cu $S/k_select.cu $S/k_cache.cu $S/k_ffn.cu \
  $S/k_reduce.cu $S/k_decode.cu $S/store.cu -ldl -lpthread
