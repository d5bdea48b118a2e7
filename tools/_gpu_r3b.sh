#!/bin/bash
# C2 phase trace of the current edge kernel: headline (round-robin) mode and one cold step
mkdir -p gpurun_out
timeout 600 python tools/trace_phases.py --config c2 --rr 23 --reps 2 > gpurun_out/r3b_trace_rr.txt 2>&1
timeout 600 python tools/trace_phases.py --config c2 --reps 2 > gpurun_out/r3b_trace_cold.txt 2>&1
