#!/bin/bash
# 16-byte finalise records (EPG_FIN_REC16=0: the 32-byte records): A/B on C3 and C2, tests
mkdir -p gpurun_out
for R in 1 0; do
  EPG_FIN_REC16=$R timeout 900 python tools/c3_step.py > gpurun_out/r2q_c3_r$R.json 2> gpurun_out/r2q_c3_r$R.err
  EPG_FIN_REC16=$R timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2q_c2_r$R.json 2> gpurun_out/r2q_c2_r$R.err
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2q_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2q_tests.log
