timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_edge_occ' -c 1 -o gpurun_out/full_c3_g python tools/ncu_variants.py --config c3 --reps 1 --variants rb > gpurun_out/full_c3_g.log 2>&1
ncu -i gpurun_out/full_c3_g.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/mix_c3_g.csv 2>&1
ncu -i gpurun_out/full_c3_g.ncu-rep --page details > gpurun_out/full_c3_g.txt 2>&1
gzip -f gpurun_out/mix_c3_g.csv
rm -f gpurun_out/full_c3_g.ncu-rep
