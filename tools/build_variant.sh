#!/usr/bin/env bash
# Builds libifa_b200.so with extra -D switches into build/<name>/ for A/B
# timing (load it with IFA_B200_LIB=build/<name>/libifa_b200.so).
#   tools/build_variant.sh NAME -DIFA_QUAD_MAGIC_S=0 ...
set -eu
NAME=$1; shift
mkdir -p build/$NAME
C=paper_2409_16997_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -shared -o build/$NAME/libifa_b200.so \
  $C/abi.cu $C/host_abi.cu $C/attn.cu $C/attn_half.cu $C/attn_pp.cu $C/attn_ws.cu $C/quant.cu $C/code_bounds.cpp $C/tensor_io.cpp -lcuda
