#!/bin/bash
# pre-wait L2 prefetch on the first step of a call only: GPU suite, C2 A/B, C3 step
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3n_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3n_tests.log
for i in 1 2; do
  for v in 0 1; do
    echo "pf$v $(EPG_PREWAIT_PF=$v timeout 600 python bench.py --no-cpu-baseline --no-comparators --no-c3 2>/dev/null | tail -1)"
  done
done > gpurun_out/r3n.txt
timeout 900 python tools/c3_step.py > gpurun_out/r3n_c3.json 2>/dev/null
