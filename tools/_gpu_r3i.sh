#!/bin/bash
# E from registers in the owned-row update: GPU suite, C2 / C3 A/B against fc575ef's predecessor build
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3i_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3i_tests.log
for v in base new base new; do
  if [ $v = base ]; then export EPG_LIB_PATH=$PWD/tools/_trace/libepg_base.so; else unset EPG_LIB_PATH; fi
  timeout 900 python tools/c3_step.py >> gpurun_out/r3i_c3_$v.jsonl 2>/dev/null
done
unset EPG_LIB_PATH
timeout 600 python bench.py --no-cpu-baseline --no-comparators --no-c3 > gpurun_out/r3i_c2_new.json 2>/dev/null
