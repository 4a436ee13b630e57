# Build a tuning variant differing only in pf_stokes.cu macros: tools/variant_stokes.sh NAME -DMACRO=V ...
set -e
B=paper_2312_15554_b200/build
name=$1; shift
mkdir -p $B/v_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-O3 -I include -DNDEBUG -Xptxas -v "$@" -c paper_2312_15554_b200/csrc/pf_stokes.cu -o $B/v_$name/pf_stokes.o 2> $B/v_$name/ptxas.txt
objs=$(ls $B/*.o | grep -v pf_stokes.o)
nvcc -shared -o $B/lib_$name.so $objs $B/v_$name/pf_stokes.o -gencode arch=compute_100a,code=sm_100a -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath,/usr/local/cuda/lib64
echo built $name
