#!/bin/bash
# DEVELOPMENT: build libutf8v_cuda.so variants with extra -D flags for one
# source file: tools/kvar.sh SRC NAME "-DFLAG ..." -> build/var_NAME/libutf8v_cuda.so
set -e
cd "$(dirname "$0")/.."
src=$1; name=$2; shift 2
out=build/var_$name; mkdir -p $out
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 -Iinclude --expt-relaxed-constexpr"
nvcc $A $@ -c paper_2010_03090_b200/csrc/$src -o $out/$src.o
objs=$(ls build/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libutf8v_cuda.so $out/$src.o $objs -lcudart
echo $out/libutf8v_cuda.so
