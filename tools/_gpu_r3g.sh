#!/bin/bash
# C2 step experiments: finalise CTA size, finalise late trigger, edge kernel staging after the PDL wait
mkdir -p gpurun_out
run() { timeout 600 env "$@" python bench.py --no-cpu-baseline --no-comparators --no-c3 2>/dev/null | tail -1; }
for i in 1 2; do
  echo "base $(run X=1)"
  echo "fin128 $(run EPG_FIN_THREADS=128)"
  echo "fin64 $(run EPG_FIN_THREADS=64)"
  echo "finlate $(run EPG_FIN_LATE=1)"
  echo "latestage $(run EPG_EDGE_LATE_STAGE=1)"
done > gpurun_out/r3g.txt
