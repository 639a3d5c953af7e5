#!/bin/bash
# Build an experimental variant of libgzb200.so: tools/build_variant.sh NAME [-DFLAG=V ...]
# Output: build/var/NAME/libgzb200.so (load it with GZ_LIB=...).  GZ_SRC: alternate
# source root (default: this checkout).
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
src=${GZ_SRC:-$root}
out=$root/build/var/$name
mkdir -p "$out"
cd "$src/paper_2405_19493_b200/csrc"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xptxas -v \
  -Xcompiler -fPIC,-ffp-contract=off,-O2 -ccbin /usr/bin/g++ "$@" -shared -o "$out/libgzb200.so" gz_engine.cu gz_verify.cu 2> "$out/ptxas.log" || { grep -B3 error "$out/ptxas.log" | head; exit 1; }
grep -A3 'k_polar_qILi0' "$out/ptxas.log" | grep -E 'registers|spill' | tr '\n' ' '; echo " [$name]"
