#!/bin/bash
# C2 with the 768-row execution cap against 704
mkdir -p gpurun_out
for r in 704 768 704 768; do
  echo "rows$r $(timeout 600 python bench.py --no-cpu-baseline --no-comparators --no-c3 --exec-rows $r 2>/dev/null | tail -1)" >> gpurun_out/r3y.txt
done
