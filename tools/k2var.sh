#!/bin/bash
# DEVELOPMENT: build libutf8v_cuda.so variants with extra -D flags for batch.cu
# experiments: tools/k2var.sh NAME "-DFLAG ..."  ->  build/var_NAME/libutf8v_cuda.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/var_$name; mkdir -p $out
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 -Iinclude --expt-relaxed-constexpr"
nvcc $A $@ -c paper_2010_03090_b200/csrc/batch.cu -o $out/batch.cu.o
objs=$(ls build/*.o | grep -v batch.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libutf8v_cuda.so $out/batch.cu.o $objs -lcudart
echo $out/libutf8v_cuda.so
