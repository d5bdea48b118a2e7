#!/bin/bash
# lo/hi halo landing + 16-byte finalise records + FTZ MUFU: tests, C3 step, C2 bench (x2), C5
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2s_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2s_tests.log
timeout 900 python tools/c3_step.py > gpurun_out/r2s_c3.json 2> gpurun_out/r2s_c3.err
for i in 1 2; do timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators >> gpurun_out/r2s_c2.jsonl 2>> gpurun_out/r2s_c2.err; done
timeout 1200 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --no-comparators > gpurun_out/r2s_c5.json 2> gpurun_out/r2s_c5.err
