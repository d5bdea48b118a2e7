#!/bin/bash
# class-split finalise records: tests, C3 step, C2 bench, round-robin trace of C2
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2l_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2l_tests.log
timeout 900 python tools/c3_step.py > gpurun_out/r2l_c3.json 2> gpurun_out/r2l_c3.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2l_c2.json 2> gpurun_out/r2l_c2.err
timeout 600 python tools/trace_phases.py --config c2 --rr 23 --reps 2 > gpurun_out/r2l_trace_rr.txt 2>&1
