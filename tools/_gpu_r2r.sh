#!/bin/bash
# TMA bulk copies for early halo rows: tests, C3 step, C2 bench, C3 ncu
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2r_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2r_tests.log
timeout 900 python tools/c3_step.py > gpurun_out/r2r_c3.json 2> gpurun_out/r2r_c3.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/r2r_c2.json 2> gpurun_out/r2r_c2.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o gpurun_out/r2r_edge_c3 \
    python tools/ncu_variants.py --config c3 --reps 1 --variants rb > /dev/null 2>&1
ncu -i gpurun_out/r2r_edge_c3.ncu-rep --page raw --csv > gpurun_out/r2r_raw_edge_c3.csv 2>&1
ncu -i gpurun_out/r2r_edge_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/r2r_sass_edge_c3.csv 2>&1
ncu -i gpurun_out/r2r_edge_c3.ncu-rep --page details > gpurun_out/r2r_details_edge_c3.txt 2>&1
gzip -f gpurun_out/r2r_raw_edge_c3.csv gpurun_out/r2r_sass_edge_c3.csv; rm -f gpurun_out/r2r_edge_c3.ncu-rep
for sc in c1_single c1_multiwave sharded; do
  timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py $sc > gpurun_out/r2r_san_racecheck_$sc.log 2>&1
  timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py $sc > gpurun_out/r2r_san_synccheck_$sc.log 2>&1
done
