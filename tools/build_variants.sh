#!/bin/bash
# Measurement builds of libhm_page.so with compile-time switches, loaded with
# HM_LIB_VARIANT=<name> (paper_2303_02868_b200/_native.py).  Usage:
#   tools/build_variants.sh name "-DFLAG=1 -DOTHER=2" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
PKG=paper_2303_02868_b200
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  obj=$PKG/_obj_$name; mkdir -p $obj
  for src in hm_error.cpp pagetable.cpp page_adam.cu page_adam_tma.cu page_kernels.cu page_dp.cu page_dp_onepass.cu; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC \
      -Xcompiler -O3 --expt-relaxed-constexpr $flags -I include -c $PKG/csrc/$src -o $obj/${src%.*}.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $PKG/libhm_page_$name.so $obj/*.o
  echo "built $PKG/libhm_page_$name.so ($flags)"
done
