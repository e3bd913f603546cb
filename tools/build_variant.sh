#!/bin/bash
# build an experimental variant of librecoil.so: tools/build_variant.sh OUT.so [-DFLAG=...]
# SRC=path/to/decode.cu overrides the kernel source (default: the tree's decode.cu)
OUT=$1; shift
SRC=${SRC:-paper_2306_12141_b200/csrc/kernels/decode.cu}
cd "$(dirname "$0")/.." && mkdir -p build_var
rm -f build_var/decode_var.o; /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2306_12141_b200/csrc/kernels "$@" -c $SRC -o build_var/decode_var.o
rm -f $OUT; [ -f build_var/decode_var.o ] && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT build_var/decode_var.o paper_2306_12141_b200/build/*.cpp.o $(ls paper_2306_12141_b200/build/*.cu.o | grep -v "/decode.cu.o") -lpthread -ldl
