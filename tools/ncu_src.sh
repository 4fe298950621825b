#!/bin/bash
# ncu --set full capture of one C2 layer launch + its SASS source page (GPU box)
tag=${1:-v9}
WHICH=query REPS=2 ncu --set full --import-source on --clock-control none -k regex:louver_layer_v9 -s 1 -c 1 -o gpurun_out/${tag}_full python tools/profile_layer.py > gpurun_out/ncu_${tag}.log 2>&1
ncu -i gpurun_out/${tag}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_src.csv 2>/dev/null
