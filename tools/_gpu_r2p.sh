#!/bin/bash
# contiguous 16-byte halo landing: tests, C3 step, C2 bench, C3 ncu source capture
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_launch_paths.py tests/test_gpu_epg2.py tests/test_gpu_rb.py -x -q > gpurun_out/r2p_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2p_tests.log
timeout 900 python tools/c3_step.py > gpurun_out/r2p_c3.json 2> gpurun_out/r2p_c3.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2p_c2.json 2> gpurun_out/r2p_c2.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o gpurun_out/r2p_edge_c3 \
    python tools/ncu_variants.py --config c3 --reps 1 --variants rb > /dev/null 2>&1
ncu -i gpurun_out/r2p_edge_c3.ncu-rep --page raw --csv > gpurun_out/r2p_raw_edge_c3.csv 2>&1
ncu -i gpurun_out/r2p_edge_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/r2p_sass_edge_c3.csv 2>&1
ncu -i gpurun_out/r2p_edge_c3.ncu-rep --page details > gpurun_out/r2p_details_edge_c3.txt 2>&1
gzip -f gpurun_out/r2p_raw_edge_c3.csv gpurun_out/r2p_sass_edge_c3.csv; rm -f gpurun_out/r2p_edge_c3.ncu-rep
