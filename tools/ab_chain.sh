# A/B of general diffeo chains (twist o bend, with / without the 100k mesh) under gpurun
cd ${GRAFT_REPO_ROOT:-.}
python - <<'PY'
import json
d = json.load(open("configs/c4_twist_bend_mesh_1080p.json"))
d["scene"]["primitives"] = [p for p in d["scene"]["primitives"] if p["kind"] != "mesh"]
json.dump(d, open("/tmp/c4_twist_bend_1080p.json", "w"))
PY
echo "== default"; python tools/prof_frame.py configs/c4_twist_bend_mesh_1080p.json /tmp/c4_twist_bend_1080p.json --frames 5 --warmup 1 --time
for v in build/exp/librray_*.so; do
  echo "== $(basename $v .so)"
  RRAY_CUDA_LIB=$PWD/$v python tools/prof_frame.py configs/c4_twist_bend_mesh_1080p.json /tmp/c4_twist_bend_1080p.json --frames 5 --warmup 1 --time
done
