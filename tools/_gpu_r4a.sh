#!/bin/bash
# 768-row execution cap: GPU suite, then the final evidence (bench lines + ncu) of the round's last build
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r4a_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r4a_tests.log
bash tools/_gpu_r3z.sh
