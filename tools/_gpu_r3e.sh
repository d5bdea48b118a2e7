#!/bin/bash
# one-wave epg_run_edges ranges trigger PDL early: GPU suite, C2 A/B vs the previous build, trace
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3e_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3e_tests.log
for i in 1 2; do
  for v in base new; do
    if [ $v = base ]; then export EPG_LIB_PATH=$PWD/tools/_trace/libepg_base.so; else unset EPG_LIB_PATH; fi
    timeout 600 python bench.py --no-cpu-baseline --no-comparators --no-c3 > gpurun_out/r3e_c2_${v}_$i.json 2>/dev/null
  done
done
unset EPG_LIB_PATH
timeout 900 python bench.py > gpurun_out/r3e_bench_full.json 2> gpurun_out/r3e_bench_full.err
