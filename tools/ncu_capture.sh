#!/bin/bash
# ncu --set full capture of the first march2/march kernel launch of one frame,
# exported on the GPU box to CSV (raw metrics, details, per-line source+SASS)
# so that only small files come back:  tools/ncu_capture.sh NAME CONFIG [KERNEL_REGEX]
cd "$(dirname "$0")/.."
name=$1; cfg=$2; kre=${3:-regex:march2?_kernel}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k "$kre" -c 1 \
  -o /tmp/$name python tools/prof_frame.py "$cfg" --frames 1 > gpurun_out/ncu_$name.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_src.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>/dev/null
gzip -f gpurun_out/${name}_src.csv gpurun_out/${name}_sass.csv
rm -f /tmp/$name.ncu-rep
