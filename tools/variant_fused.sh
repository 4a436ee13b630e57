#!/bin/bash
# Build a tuning variant of the library that differs only in pf_fused.cu's macros:
#   tools/variant_fused.sh NAME -DMACRO=VALUE ...   -> paper_2312_15554_b200/build/lib_NAME.so
# (the other objects come from the product build in paper_2312_15554_b200/build/)
set -e
name=$1; shift
B=paper_2312_15554_b200/build
mkdir -p $B/v_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=true -std=c++17 -Xcompiler -fPIC,-O3 \
  -I include -Xptxas -v -DNDEBUG "$@" -c paper_2312_15554_b200/csrc/pf_fused.cu -o $B/v_$name/pf_fused.o \
  2> $B/v_$name/pf_fused.ptxas.txt
objs=$(ls $B/*.o | grep -v pf_fused.o)
nvcc -shared -o $B/lib_$name.so $objs $B/v_$name/pf_fused.o -gencode arch=compute_100a,code=sm_100a \
  -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath,/usr/local/cuda/lib64
echo built $B/lib_$name.so
