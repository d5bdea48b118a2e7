#!/bin/bash
# final bench line of the round's last build
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final3_bench_c2.json 2> gpurun_out/final3_bench_c2.err
echo "rc=$?" >> gpurun_out/final3_bench_c2.err
