#!/bin/bash
# C2 trace: edge kernel + finalise of one round-robin step, and finalise -> next edge kernel
mkdir -p gpurun_out
timeout 600 python tools/trace_phases.py --config c2 --rr 23 --reps 2 > gpurun_out/r3f_trace_rr.txt 2>&1
timeout 600 python tools/trace_phases.py --config c2 --rr 23 --reps 2 --chain > gpurun_out/r3f_trace_chain.txt 2>&1
