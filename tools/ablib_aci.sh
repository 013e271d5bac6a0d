#!/bin/bash
# A/B library: recompile aci.cu with extra -D flags, link with the in-tree gemm.cu/prrlu.cu objects
# usage: tools/ablib_aci.sh NAME [-DFOO=1 ...]   -> tools/libab/libaci_NAME.so
set -e
name=$1; shift
mkdir -p tools/libab
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include"
nvcc $F "$@" -c -o tools/libab/aci_$name.o paper_2604_00037_b200/csrc/aci.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libab/libaci_$name.so tools/libab/aci_$name.o paper_2604_00037_b200/build/gemm.cu.o paper_2604_00037_b200/build/prrlu.cu.o -lcudart
