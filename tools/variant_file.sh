#!/bin/bash
# Build a tuning variant of the library differing only in one source file's macros:
#   tools/variant_file.sh SRC.cu NAME -DMACRO=VALUE ...   -> paper_2312_15554_b200/build/lib_NAME.so
# (the other objects come from the product build in paper_2312_15554_b200/build/)
set -e
src=$1; name=$2; shift 2
B=paper_2312_15554_b200/build
obj=$(basename $src .cu).o
fmad=false; case $src in pf_fused.cu|pf_fused_transport.cu) fmad=true;; esac
mkdir -p $B/v_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=$fmad -std=c++17 -Xcompiler -fPIC,-O3 \
  -I include -Xptxas -v -DNDEBUG "$@" -c paper_2312_15554_b200/csrc/$src -o $B/v_$name/$obj 2> $B/v_$name/ptxas.txt
objs=$(ls $B/*.o | grep -v "/$obj")
nvcc -shared -o $B/lib_$name.so $objs $B/v_$name/$obj -gencode arch=compute_100a,code=sm_100a \
  -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath,/usr/local/cuda/lib64
echo built $name
