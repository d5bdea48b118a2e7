#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3t_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3t_tests.log
