#!/bin/bash
# A/B library: recompile gemm.cu with extra -D flags, link with the in-tree aci.cu/prrlu.cu objects
# usage: tools/ablib_gemm.sh NAME [-DFOO=1 ...]   -> tools/libab/libaci_NAME.so
set -e
name=$1; shift
mkdir -p tools/libab
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include"
nvcc $F "$@" -Xptxas -v -c -o tools/libab/gemm_$name.o paper_2604_00037_b200/csrc/gemm.cu 2> tools/libab/ptxas_$name.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libab/libaci_$name.so paper_2604_00037_b200/build/aci.cu.o tools/libab/gemm_$name.o paper_2604_00037_b200/build/prrlu.cu.o -lcudart
