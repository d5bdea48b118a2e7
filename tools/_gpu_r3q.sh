#!/bin/bash
# smoke() of the final build, C3 step record (tools/c3_step.py, with comparators)
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3q_smoke.txt 2>&1
echo "rc=$?" >> gpurun_out/r3q_smoke.txt
timeout 1500 python tools/c3_step.py --comparators > gpurun_out/r3q_c3.json 2> gpurun_out/r3q_c3.err
