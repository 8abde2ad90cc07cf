# A/B of build/exp variants on C3 (unlit + lit) timing and full-frame parity under gpurun
cd ${GRAFT_REPO_ROOT:-.}
echo "== default"; python tools/prof_frame.py configs/c3_bumps16_1080p.json configs/c3_bumps16_shadows_1080p.json --frames 10 --warmup 2 --time
for v in build/exp/librray_*.so; do
  n=$(basename $v .so)
  echo "== $n"
  RRAY_CUDA_LIB=$PWD/$v python tools/prof_frame.py configs/c3_bumps16_1080p.json configs/c3_bumps16_shadows_1080p.json --frames 10 --warmup 2 --time
  RRAY_CUDA_LIB=$PWD/$v RR_PARITY_LOG=gpurun_out/parity_$n.jsonl python -m pytest tests/test_gpu_frame_parity.py -q -p no:cacheprovider -k "c3_1080p_full or c5_4k" --timeout 900 2>&1 | tail -1
  cat gpurun_out/parity_$n.jsonl
done
