#!/bin/bash
# C3 occupancy experiments: P = 1024 / 768 with 4 or 5 resident CTAs per SM
mkdir -p gpurun_out
timeout 600 python tools/c3_step.py > gpurun_out/r2e_c3_p1024.json 2> gpurun_out/r2e_c3_p1024.err
timeout 600 python tools/c3_step.py --part-size 768 --exec-rows 560 > gpurun_out/r2e_c3_p768.json 2> gpurun_out/r2e_c3_p768.err
EPG_LIB_PATH=tools/_trace/libepg_minb5.so timeout 600 python tools/c3_step.py --part-size 768 --exec-rows 560 > gpurun_out/r2e_c3_p768_m5.json 2> gpurun_out/r2e_c3_p768_m5.err
EPG_LIB_PATH=tools/_trace/libepg_minb5.so timeout 600 python tools/c3_step.py --part-size 896 --exec-rows 560 > gpurun_out/r2e_c3_p896_m5.json 2> gpurun_out/r2e_c3_p896_m5.err
EPG_GRAPHS=0 timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2e_bench_nograph.json 2> gpurun_out/r2e_bench_nograph.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2e_bench_graph.json 2> gpurun_out/r2e_bench_graph.err
