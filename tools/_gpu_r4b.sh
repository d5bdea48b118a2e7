#!/bin/bash
# final tree: smoke() and the GPU suite
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4b_smoke.txt 2>&1
echo "rc=$?" >> gpurun_out/r4b_smoke.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r4b_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r4b_tests.log
