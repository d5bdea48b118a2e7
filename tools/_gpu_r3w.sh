#!/bin/bash
# C3 execution row cap sweep with the current kernel (R3: 704 rows is the default)
mkdir -p gpurun_out
for r in 704 672 736 704 768; do
  echo "rows$r $(timeout 900 python tools/c3_step.py --exec-rows $r 2>/dev/null | tail -1)" >> gpurun_out/r3w.txt
done
