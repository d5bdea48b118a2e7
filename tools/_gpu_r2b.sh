#!/bin/bash
# source-level ncu captures of the staged edge kernel (C2 and C3, EPG-RB map in growth order)
mkdir -p gpurun_out
for CFG in c2 c3; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'k_edge_occ' -c 1 \
      -o gpurun_out/src_$CFG python tools/ncu_variants.py --config $CFG --reps 1 --variants rb > gpurun_out/src_$CFG.log 2>&1
  ncu -i gpurun_out/src_$CFG.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$CFG.csv 2>&1
  ncu -i gpurun_out/src_$CFG.ncu-rep --page source --csv --print-source cuda > gpurun_out/cuda_$CFG.csv 2>&1
  ncu -i gpurun_out/src_$CFG.ncu-rep --page details > gpurun_out/details_$CFG.txt 2>&1
  gzip -f gpurun_out/sass_$CFG.csv gpurun_out/cuda_$CFG.csv
  rm -f gpurun_out/src_$CFG.ncu-rep
done
