#!/bin/bash
# SoA derived records + pointer-based Phi_4: GPU suite, then C2 / C3 A/B against the previous build
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3d_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3d_tests.log
for i in 1 2; do
  for v in base new; do
    if [ $v = base ]; then export EPG_LIB_PATH=$PWD/tools/_trace/libepg_base.so; else unset EPG_LIB_PATH; fi
    timeout 600 python bench.py --no-cpu-baseline --no-comparators --no-c3 > gpurun_out/r3d_c2_${v}_$i.json 2>/dev/null
  done
done
for v in base new; do
  if [ $v = base ]; then export EPG_LIB_PATH=$PWD/tools/_trace/libepg_base.so; else unset EPG_LIB_PATH; fi
  timeout 900 python tools/c3_step.py > gpurun_out/r3d_c3_$v.json 2> gpurun_out/r3d_c3_$v.err
done
