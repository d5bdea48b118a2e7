#!/bin/bash
# direct one-step launches + segmented-scan reduce: full GPU tests, default bench, C4 bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_tests.log
timeout 1500 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_c4.json 2> gpurun_out/r2f_bench_c4.err
