#!/bin/bash
# Development: the out-of-line GEMM experiment (csrc/gemm_bal.cu, -rdc, one
# gemm_bal_x for every kernel) into variants/librnntg_ext.so.
set -e
cd "$(dirname "$0")/../paper_2211_00484_b200"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -rdc=true -DRNNTG_GEMM_EXTERN"
O=$(mktemp -d)
for f in capi gemm_exact decode fsa cluster debug; do nvcc $F -c csrc/$f.cu -o $O/$f.o & done
nvcc $F -maxrregcount=128 -c csrc/gemm_bal.cu -o $O/gemm_bal.o
wait
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -rdc=true -o variants/librnntg_ext.so $O/*.o
rm -rf "$O"
