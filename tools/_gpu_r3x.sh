#!/bin/bash
# C3 execution row cap sweep, larger caps (each twice)
mkdir -p gpurun_out
for r in 768 832 896 960 768 832 896 960; do
  echo "rows$r $(timeout 900 python tools/c3_step.py --exec-rows $r 2>/dev/null | tail -1)" >> gpurun_out/r3x.txt
done
