#!/bin/bash
# Development: build librnntg.so with extra nvcc flags into
# paper_2211_00484_b200/variants/librnntg_<name>.so (load with RNNTG_LIB=...).
# usage: tools/build_variant.sh <name> [nvcc flags...]
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2211_00484_b200"
mkdir -p variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared \
  -cudart shared "$@" -o variants/librnntg_$name.so csrc/capi.cu csrc/gemm_exact.cu csrc/decode.cu csrc/fsa.cu \
  csrc/logadd.cu csrc/cluster.cu csrc/debug.cu csrc/synth.cpp
python ../tools/fadd_dist.py variants/librnntg_$name.so beam_kernelILi4ELb0ELb0 100 | sed "s/^/[$name] /"
