# A/B of build/exp variants on the C3 and C3 + 2 lights frames under gpurun
# (alternated twice; frame digests printed for bit-identity checks)
cd ${GRAFT_REPO_ROOT:-.}
CFGS=${AB_CFGS:-"configs/c3_bumps16_1080p.json configs/c3_bumps16_shadows_1080p.json"}
for rep in 1 2; do
  echo "== default"; python tools/prof_frame.py $CFGS --frames 10 --warmup 2 --time
  for v in build/exp/librray_*.so; do
    echo "== $(basename $v .so)"
    RRAY_CUDA_LIB=$PWD/$v python tools/prof_frame.py $CFGS --frames 10 --warmup 2 --time
  done
done
