#!/bin/bash
# pre-wait L2 prefetch of the state rows (single-wave grids): C2 A/B (EPG_PREWAIT_PF=0/1), trace
mkdir -p gpurun_out
for i in 1 2; do
  for v in 0 1; do
    echo "pf$v $(EPG_PREWAIT_PF=$v timeout 600 python bench.py --no-cpu-baseline --no-comparators --no-c3 2>/dev/null | tail -1)"
  done
done > gpurun_out/r3m.txt
EPG_PREWAIT_PF=1 timeout 600 python tools/trace_phases.py --config c2 --rr 23 --reps 1 --chain > gpurun_out/r3m_trace.txt 2>&1
