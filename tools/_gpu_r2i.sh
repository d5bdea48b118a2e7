#!/bin/bash
# GPU placement kernel: tests, C3 / C2 timing, sanitizers on the new paths
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_tests.log
B="--no-c3 --no-cpu-baseline --no-comparators"
timeout 900 python tools/c3_step.py > gpurun_out/r2i_c3.json 2> gpurun_out/r2i_c3.err
timeout 900 python bench.py $B > gpurun_out/r2i_c2_p1032.json 2> gpurun_out/r2i_c2_p1032.err
timeout 900 python bench.py $B --part-size 1024 > gpurun_out/r2i_c2_p1024.json 2> gpurun_out/r2i_c2_p1024.err
for t in memcheck racecheck synccheck; do
  for sc in c1_single c1_multiwave wide hub spmv sharded; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py $sc > gpurun_out/san_${t}_${sc}.log 2>&1
  done
done
