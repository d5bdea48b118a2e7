#!/bin/bash
# final round-2 evidence for the current build: bench lines (C2 + C3 sub-record, reference arm,
# C4, C5), C2 launch list, per-schedule traffic (C2, C3), full captures of the edge kernel and the
# finalise (C2, C3)
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python bench.py > $OUT/final_bench_c2.json 2> $OUT/final_bench_c2.err
timeout 900 python bench.py --impl reference > $OUT/final_bench_ref.json 2> $OUT/final_bench_ref.err
timeout 1200 python bench.py --config c4 --no-cpu-baseline > $OUT/final_bench_c4.json 2> $OUT/final_bench_c4.err
timeout 900 python bench.py --config c5 --no-cpu-baseline > $OUT/final_bench_c5.json 2> $OUT/final_bench_c5.err
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-comparators --no-c3 > $OUT/launches_c2.log 2>&1
for CFG in c2 c3; do
  V=rb,default,naive; [ $CFG = c3 ] && V=rb,default
  timeout 1500 ncu --metrics $M --csv --log-file $OUT/variants_$CFG.csv -k regex:'^(k_edge_occ|k_finalise_rec|k_finalise_rec16|k_finalise3|k_naive_edges|k_naive_update)$' \
      python tools/ncu_variants.py --config $CFG --reps 1 --variants $V > $OUT/variants_$CFG.log 2>&1
  for K in edge fin; do
    R='k_edge_occ'; [ $K = fin ] && R='^k_finalise_rec16$'
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$R -c 1 -o $OUT/full_${K}_$CFG \
        python tools/ncu_variants.py --config $CFG --reps 1 --variants rb > /dev/null 2>&1
    ncu -i $OUT/full_${K}_$CFG.ncu-rep --page details > $OUT/details_${K}_$CFG.txt 2>&1
    ncu -i $OUT/full_${K}_$CFG.ncu-rep --page raw --csv > $OUT/raw_${K}_$CFG.csv 2>&1
    ncu -i $OUT/full_${K}_$CFG.ncu-rep --page source --csv --print-source sass > $OUT/sass_${K}_$CFG.csv 2>&1
    gzip -f $OUT/raw_${K}_$CFG.csv $OUT/sass_${K}_$CFG.csv
    [ $K = fin ] && rm -f $OUT/full_${K}_$CFG.ncu-rep
  done
done
ls -la $OUT
