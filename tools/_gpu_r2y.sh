#!/bin/bash
# EPG-RB leaf size on C3: partition time vs replication vs step
mkdir -p gpurun_out
for LP in 512 1024 2048 4096; do
  timeout 900 python tools/c3_step.py --leaf-parts $LP > gpurun_out/r2y_c3_lp$LP.json 2> gpurun_out/r2y_c3_lp$LP.err
done
