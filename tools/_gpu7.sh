timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_edge_occ' -c 1 -o gpurun_out/full_c3_r2e python tools/ncu_variants.py --config c3 --reps 1 --variants rb > gpurun_out/full_c3_r2e.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_finalise_rec<' -c 1 -o gpurun_out/full_c3_r2f python tools/ncu_variants.py --config c3 --reps 1 --variants rb > gpurun_out/full_c3_r2f.log 2>&1
ls -la gpurun_out/full_c3_r2*
