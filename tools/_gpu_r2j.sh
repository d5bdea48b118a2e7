#!/bin/bash
# warp-cooperative placement: tests, C3 remap time, C2 / C5 bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2j_tests.log
timeout 900 python tools/c3_step.py > gpurun_out/r2j_c3.json 2> gpurun_out/r2j_c3.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2j_c2.json 2> gpurun_out/r2j_c2.err
timeout 1200 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_c5.json 2> gpurun_out/r2j_c5.err
EPG_PLACE=0 timeout 1200 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --no-comparators > gpurun_out/r2j_c5_noplace.json 2> gpurun_out/r2j_c5_noplace.err
