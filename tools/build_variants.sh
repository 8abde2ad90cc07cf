#!/bin/bash
# Builds experimental variants of librray_cuda.so into build/exp/ for A/B
# timing on the GPU box (RRAY_CUDA_LIB=... python bench.py, tools/ab.sh).
# Variants compile in parallel, each in its own scratch copy of csrc/.
#   tools/build_variants.sh name "-DMACRO=1 ..." [name "flags"]...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CSRC=$ROOT/paper_2005_05386_b200/csrc
mkdir -p "$ROOT/build/exp"
pids=()
names=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  d=$(mktemp -d /tmp/rrvar_XXXX)
  mkdir -p "$d/paper_2005_05386_b200" && cp -r "$CSRC" "$d/paper_2005_05386_b200/csrc" && cp -r "$ROOT/include" "$d/include"
  ( cd "$d/paper_2005_05386_b200/csrc" && make -s clean >/dev/null &&
    make -s -j6 EXTRA_NVFLAGS="$flags" >/dev/null 2>&1 &&
    cp librray_cuda.so "$ROOT/build/exp/librray_$name.so" &&
    echo "$name: built" ; rm -rf "$d" ) &
  pids+=($!)
  names+=($name)
done
for p in "${pids[@]}"; do wait $p; done
