#!/bin/bash
# build an experimental variant of librecoil.so: tools/build_variant.sh OUT.so -DFLAG=...
OUT=$1; shift
cd "$(dirname "$0")/.." && mkdir -p build_var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Iinclude "$@" -c paper_2306_12141_b200/csrc/kernels/decode.cu -o build_var/decode_var.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT build_var/decode_var.o paper_2306_12141_b200/build/*.cpp.o -lpthread
