#!/bin/bash
# final C2 evidence of the current build: bench line (with C3 sub-record), launch list, full capture
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python bench.py > $OUT/final2_bench_c2.json 2> $OUT/final2_bench_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-comparators --no-c3 > $OUT/launches_c2.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 1500 ncu --metrics $M --csv --log-file $OUT/variants_c2.csv -k regex:'^(k_edge_occ|k_finalise_rec|k_finalise_rec16|k_finalise3|k_naive_edges|k_naive_update)$' \
    python tools/ncu_variants.py --config c2 --reps 1 --variants rb,default,naive > $OUT/variants_c2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o $OUT/full_edge_c2 \
    python tools/ncu_variants.py --config c2 --reps 1 --variants rb > /dev/null 2>&1
ncu -i $OUT/full_edge_c2.ncu-rep --page source --csv --print-source sass > $OUT/sass_edge_c2.csv 2>&1
gzip -f $OUT/sass_edge_c2.csv
