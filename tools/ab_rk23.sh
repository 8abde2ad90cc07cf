# A/B of build/exp variants on the C3 rk23 frame under gpurun (alternated twice)
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2; do
  echo "== default"; python tools/prof_frame.py configs/c3_bumps16_rk23_1080p.json configs/c3_bumps16_1080p.json --frames 10 --warmup 2 --time
  for v in build/exp/librray_*.so; do
    echo "== $(basename $v .so)"
    RRAY_CUDA_LIB=$PWD/$v python tools/prof_frame.py configs/c3_bumps16_rk23_1080p.json --frames 10 --warmup 2 --time
  done
done
