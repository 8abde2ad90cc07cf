#!/bin/bash
# A/B timing of build/exp/librray_*.so variants on the GPU box (run under gpurun).
cd "$(dirname "$0")/.."
# Either A/B library variants (default) or option sets: tools/ab.sh --opts "cull_grid=32" "cull_grid=64"
# (AB_ARGS="--opt cull_radius_sigma=5.5" adds bench options to every library run)
if [ "$1" = "--opts" ]; then
  shift
  variants=("$@")
  mode=opts
else
  variants=(build/exp/librray_*.so)
  mode=libs
fi
for v in "${variants[@]}"; do
  if [ $mode = libs ]; then
    name=$(basename $v .so)
    RRAY_CUDA_LIB=$PWD/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras $AB_ARGS > gpurun_out/ab_$name.log 2>&1
  else
    name=$(echo "$v" | tr ' =' '_-')
    optargs=""
    for o in $v; do optargs="$optargs --opt $o"; done
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras $optargs > gpurun_out/ab_$name.log 2>&1
  fi
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{name}.log").read().strip().splitlines()[-1])
    sh = d.get("shadows") or {}
    print(f"{name:28s} ms/frame {d['ms_per_step']:8.3f} fps {d['fps']:7.2f} frac {d['roofline']['frac']:.3f} neff {d['n_eff_bumps']:.2f} clk {d['clocks']['sm_mhz']} | shadows ms {sh.get('ms_per_frame', 0):.3f} fps {sh.get('fps', 0):.1f}")
except Exception as e:
    print(name, "FAILED", e)
PY
done
