#!/bin/bash
# bank-conflict-aware placement + 288-thread VPT4: full GPU tests; A/B on C2 (P 1032 / 1024) and C3
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_tests.log
B="--no-c3 --no-cpu-baseline --no-comparators"
timeout 900 python bench.py $B > gpurun_out/r2h_c2_p1032.json 2> gpurun_out/r2h_c2_p1032.err
timeout 900 python bench.py $B --part-size 1024 > gpurun_out/r2h_c2_p1024.json 2> gpurun_out/r2h_c2_p1024.err
EPG_PLACE=0 timeout 900 python bench.py $B --part-size 1024 > gpurun_out/r2h_c2_p1024_noplace.json 2> gpurun_out/r2h_c2_p1024_noplace.err
timeout 900 python tools/c3_step.py > gpurun_out/r2h_c3.json 2> gpurun_out/r2h_c3.err
EPG_PLACE=0 timeout 900 python tools/c3_step.py > gpurun_out/r2h_c3_noplace.json 2> gpurun_out/r2h_c3_noplace.err
