#!/usr/bin/env bash
# Builds libifa_b200.so with extra -D switches into build/<name>/ for A/B
# timing (load it with IFA_B200_LIB=build/<name>/libifa_b200.so).  Only the
# translation unit SRC (default attn_pp.cu) is recompiled with the switches;
# the other objects come from the in-tree build.
#   [SRC=attn.cu] tools/build_variant.sh NAME -DIFA_PP_OBOX=0 ...
set -eu
NAME=$1; shift
SRC=${SRC:-attn_pp.cu}
cd "$(dirname "$0")/.."
make -s -j8 paper_2409_16997_b200/lib/libifa_b200.so >/dev/null
D=build/$NAME; mkdir -p $D
OBJ=paper_2409_16997_b200/lib/obj
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC --expt-relaxed-constexpr "$@" -c -o $D/$SRC.o paper_2409_16997_b200/csrc/$SRC
objs=$(ls $OBJ/*.o | grep -v "/$SRC.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libifa_b200.so $objs $D/$SRC.o -lcuda
echo $D/libifa_b200.so
