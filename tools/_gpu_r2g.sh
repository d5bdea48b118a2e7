#!/bin/bash
# 288-thread instance (C2 at P = 1032): tests + bench (no C3 / comparators), and P = 1024 for A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_launch_paths.py tests/test_gpu_parity.py -x -q > gpurun_out/r2g_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_tests.log
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2g_bench_p1032.json 2> gpurun_out/r2g_bench_p1032.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators --part-size 1024 > gpurun_out/r2g_bench_p1024.json 2> gpurun_out/r2g_bench_p1024.err
timeout 600 python tools/trace_phases.py --config c2 --part-size 1032 > gpurun_out/r2g_trace.txt 2>&1
