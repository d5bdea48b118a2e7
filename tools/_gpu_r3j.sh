#!/bin/bash
# C4 step regression hunt: 06bff80 (round-2 C4 bench build), session start (6dc33dd), current
mkdir -p gpurun_out
for v in 06bff80 base new; do
  if [ $v = new ]; then unset EPG_LIB_PATH; else export EPG_LIB_PATH=$PWD/tools/_trace/libepg_$v.so; fi
  timeout 900 python bench.py --config c4 --no-cpu-baseline --no-comparators > gpurun_out/r3j_c4_$v.json 2> gpurun_out/r3j_c4_$v.err
done
