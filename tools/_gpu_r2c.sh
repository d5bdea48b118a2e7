#!/bin/bash
# FFMA2 flux + early halo ids: parity subset, C2 bench (no C3), C3 step, C2 phase trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_epg2.py tests/test_gpu_launch_paths.py -x -q > gpurun_out/r2c_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_tests.log
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 900 python tools/c3_step.py > gpurun_out/r2c_c3.json 2> gpurun_out/r2c_c3.err
timeout 600 python tools/trace_phases.py --config c2 > gpurun_out/r2c_trace.txt 2>&1
