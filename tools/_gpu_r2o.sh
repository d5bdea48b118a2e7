#!/bin/bash
# LPT order for one-wave grids: A/B on C2, tests, trace
mkdir -p gpurun_out
B="--no-c3 --no-cpu-baseline --no-comparators"
for LPT in 1 0 1 0; do
  EPG_LPT=$LPT timeout 900 python bench.py $B >> gpurun_out/r2o_c2_lpt$LPT.jsonl 2>> gpurun_out/r2o_c2_lpt$LPT.err
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launch_paths.py tests/test_gpu_epg2.py tests/test_gpu_sharded_lib.py -x -q > gpurun_out/r2o_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2o_tests.log
timeout 900 python tools/trace_phases.py --config c2 --rr 23 --reps 2 > gpurun_out/r2o_trace_rr.txt 2>&1
