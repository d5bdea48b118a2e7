#!/bin/bash
# source-level ncu capture of the C2 edge kernel (per-SASS executed instructions + stall samples)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o gpurun_out/r3c_c2_edge \
    python tools/ncu_variants.py --config c2 --reps 1 --variants rb > gpurun_out/r3c.log 2>&1
ncu -i gpurun_out/r3c_c2_edge.ncu-rep --page source --csv --print-source sass > gpurun_out/r3c_c2_sass.csv 2>&1
ncu -i gpurun_out/r3c_c2_edge.ncu-rep --page source --csv --print-source cuda > gpurun_out/r3c_c2_cuda.csv 2>&1
ls -la gpurun_out
