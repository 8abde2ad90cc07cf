# A/B of the C4 mesh frame under gpurun: default library vs build/exp variants
cd ${GRAFT_REPO_ROOT:-.}
echo "== default"; python tools/prof_frame.py configs/c4_twist_mesh_1080p.json --frames 10 --warmup 2 --time
for v in build/exp/librray_*.so; do
  echo "== $(basename $v .so)"
  RRAY_CUDA_LIB=$PWD/$v python tools/prof_frame.py configs/c4_twist_mesh_1080p.json --frames 10 --warmup 2 --time
done
