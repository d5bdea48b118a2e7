#!/bin/bash
# re-entry check of the restored build: GPU suite + default bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r3a_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3a_tests.log
timeout 900 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err
echo "rc=$?" >> gpurun_out/r3a_bench.err
