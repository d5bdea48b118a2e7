#!/bin/bash
# ncu evidence for one round (run on the GPU box under gpurun; writes gpurun_out/).
#  1. launch list of the bench command (per-launch device time, cold/serialised)
#  2. per-variant DRAM / L2 traffic of one cfd step (EP staged, default staged, naive)
#  3. one --set full capture of the dominant kernel (k_edge_occ) and of the finalise
#  usage: tools/profile_round.sh <config> <variants for ncu_variants.py>
set -u
OUT=gpurun_out
CFG=${1:-c2}
VARS=${2:-rb,ep1,default,naive}
mkdir -p $OUT
if [ "$CFG" = "c2" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$CFG.csv \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-comparators --no-c3 > $OUT/launches_$CFG.log 2>&1
fi
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --csv --log-file $OUT/variants_$CFG.csv -k regex:'^(k_edge_occ|k_finalise_rec|k_finalise3|k_naive_edges|k_naive_update)$' \
    python tools/ncu_variants.py --config $CFG --reps 1 --variants $VARS > $OUT/variants_$CFG.log 2>&1
FIRST=${VARS%%,*}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_edge_occ -c 1 -o $OUT/full_edge_$CFG \
    python tools/ncu_variants.py --config $CFG --reps 1 --variants $FIRST > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_finalise_rec$' -c 1 -o $OUT/full_fin_$CFG \
    python tools/ncu_variants.py --config $CFG --reps 1 --variants $FIRST > /dev/null 2>&1
ls -la $OUT
