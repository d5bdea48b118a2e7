#!/bin/bash
# vectorised descriptor loads: parity subset, C3 step (x2), C2 bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_launch_paths.py -x -q > gpurun_out/r2v_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2v_tests.log
for i in 1 2; do timeout 900 python tools/c3_step.py >> gpurun_out/r2v_c3.jsonl 2>> gpurun_out/r2v_c3.err; done
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2v_c2.json 2> gpurun_out/r2v_c2.err
