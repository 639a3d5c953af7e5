#!/bin/bash
# Debug build with the in-kernel self-checks (GZ_CHECK, gz_engine.cu) for the
# compute-sanitizer stand-in runs: writes paper_2405_19493_b200/libgzb200_dbg.so;
# select it with GZ_LIB=$PWD/paper_2405_19493_b200/libgzb200_dbg.so.
set -e
cd "$(dirname "$0")/../paper_2405_19493_b200/csrc"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false \
  -DGZ_DEBUG_CHECKS -Xcompiler -fPIC,-ffp-contract=off,-O2 -ccbin /usr/bin/g++ -shared \
  -o ../libgzb200_dbg.so gz_engine.cu gz_verify.cu
