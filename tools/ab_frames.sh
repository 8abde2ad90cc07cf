#!/bin/bash
# A/B of build/exp/librray_*.so variants with tools/prof_frame.py (CUDA events,
# L2 flushed, 10 frames) on C3, C3 + 2 lights, C1.  Run under gpurun.
cd "$(dirname "$0")/.."
for v in build/exp/librray_*.so; do
  name=$(basename $v .so)
  echo "== $name"
  RRAY_CUDA_LIB=$PWD/$v timeout 300 python tools/prof_frame.py configs/c3_bumps16_1080p.json \
     configs/c3_bumps16_shadows_1080p.json configs/c1_gauss1_512.json ${AB_EXTRA_CONFIGS} --frames 10 --warmup 2 --time 2>&1 | grep -v "^$"
done
