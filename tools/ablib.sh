#!/bin/bash
# A/B library: recompile prrlu.cu with extra -D flags, link with the in-tree aci.cu/gemm.cu objects
# usage: tools/ablib.sh NAME [-DFOO=1 ...]   -> tools/libab/libaci_NAME.so
set -e
name=$1; shift
mkdir -p tools/libab
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include"
nvcc $F "$@" -c -o tools/libab/prrlu_$name.o paper_2604_00037_b200/csrc/prrlu.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libab/libaci_$name.so paper_2604_00037_b200/build/aci.cu.o paper_2604_00037_b200/build/gemm.cu.o tools/libab/prrlu_$name.o -lcudart
