#!/bin/bash
# source-level ncu captures of the current edge kernel: C3 (bandwidth regime) and C2
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o gpurun_out/r3h_c3_edge \
    python tools/ncu_variants.py --config c3 --reps 1 --variants rb > gpurun_out/r3h_c3.log 2>&1
ncu -i gpurun_out/r3h_c3_edge.ncu-rep --page source --csv --print-source sass > gpurun_out/r3h_c3_sass.csv 2>&1
ncu -i gpurun_out/r3h_c3_edge.ncu-rep --page details > gpurun_out/r3h_c3_details.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o gpurun_out/r3h_c2_edge \
    python tools/ncu_variants.py --config c2 --reps 1 --variants rb > gpurun_out/r3h_c2.log 2>&1
ncu -i gpurun_out/r3h_c2_edge.ncu-rep --page source --csv --print-source sass > gpurun_out/r3h_c2_sass.csv 2>&1
ncu -i gpurun_out/r3h_c2_edge.ncu-rep --page details > gpurun_out/r3h_c2_details.txt 2>&1
rm -f gpurun_out/*.ncu-rep
