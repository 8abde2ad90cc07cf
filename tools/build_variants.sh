#!/bin/bash
# Builds experimental variants of librray_cuda.so into build/exp/ for A/B
# timing on the GPU box (RRAY_CUDA_LIB=... python bench.py).  Usage:
#   tools/build_variants.sh name "-DMACRO=1 ..." [name "flags"]...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_2005_05386_b200/csrc
mkdir -p "$ROOT/build/exp"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -C "$CSRC" clean >/dev/null
  make -s -C "$CSRC" NVFLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I../../include -Xptxas -v $flags" >/dev/null 2>&1
  cp "$CSRC/librray_cuda.so" "$ROOT/build/exp/librray_$name.so"
  echo "$name: $(grep -A2 'ILi1ELi16ELi1E' "$CSRC/ptxas.log" | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
done
make -s -C "$CSRC" clean >/dev/null
make -s -C "$CSRC" >/dev/null 2>&1
