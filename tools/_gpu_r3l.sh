#!/bin/bash
# EPG-RB phase times on C3 (EPG_RB_TRACE), twice in one process, with the box's CPU
mkdir -p gpurun_out
( nproc; lscpu | grep -i "model name\|^CPU(s)\|Thread\|NUMA node(s)"; free -g | head -2 ) > gpurun_out/r3l_host.txt 2>&1
EPG_RB_TRACE=1 timeout 900 python tools/partition_bench.py c3 --leaf-parts 2048 2048 > gpurun_out/r3l_rb.jsonl 2> gpurun_out/r3l_rb.err
