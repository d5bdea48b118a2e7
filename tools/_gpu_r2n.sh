#!/bin/bash
# round-robin trace of C2 with finalise stamps
mkdir -p gpurun_out
timeout 900 python tools/trace_phases.py --config c2 --rr 23 --reps 2 > gpurun_out/r2n_trace_rr.txt 2>&1
timeout 600 python tools/trace_phases.py --config c2 --reps 2 > gpurun_out/r2n_trace_cold.txt 2>&1
