#!/bin/bash
# sharded overlap tests; host overhead of per-step calls; C4 ncu evidence
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded_lib.py tests/test_gpu_shard.py tests/test_gpu_parity.py -x -q > gpurun_out/r2d_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_tests.log
timeout 300 python tools/host_overhead.py > gpurun_out/r2d_host.json 2>&1
timeout 300 python tools/host_overhead.py replicas > gpurun_out/r2d_host_rep.json 2>&1
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --csv --log-file gpurun_out/variants_c4.csv -k regex:'^(k_edge_occ|k_finalise_rec|k_finalise3|k_finalise_warp|k_finalise_heavy|k_finalise_hub|k_naive_edges|k_naive_update)$' \
    python tools/ncu_variants.py --config c4 --reps 1 --variants rb,ep1,default,naive > gpurun_out/variants_c4.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o gpurun_out/full_c4 \
    python tools/ncu_variants.py --config c4 --reps 1 --variants rb > gpurun_out/full_c4.log 2>&1
ncu -i gpurun_out/full_c4.ncu-rep --page details > gpurun_out/details_c4.txt 2>&1
ncu -i gpurun_out/full_c4.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_c4.csv 2>&1
ncu -i gpurun_out/full_c4.ncu-rep --page raw --csv > gpurun_out/raw_c4.csv 2>&1
gzip -f gpurun_out/sass_c4.csv gpurun_out/raw_c4.csv
rm -f gpurun_out/full_c4.ncu-rep
