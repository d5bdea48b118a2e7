#!/bin/bash
# memory-pool release threshold: C3 setup times (partition, remap) and step with keep = 0 / 32 GiB
mkdir -p gpurun_out
for v in 0 32 0 32; do
  echo "keep$v $(EPG_POOL_KEEP_GB=$v timeout 900 python tools/c3_step.py 2>/dev/null | tail -1)" >> gpurun_out/r3s.txt
done
