#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_launch_paths.py -q > gpurun_out/r3v_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3v_tests.log
