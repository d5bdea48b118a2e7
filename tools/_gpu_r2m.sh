#!/bin/bash
# A/B of the class-split finalise records (EPG_FIN_SPLIT=0 keeps the 32-byte records)
mkdir -p gpurun_out
B="--no-c3 --no-cpu-baseline --no-comparators"
for FS in 1 0; do
  EPG_FIN_SPLIT=$FS timeout 900 python bench.py $B > gpurun_out/r2m_c2_fs$FS.json 2> gpurun_out/r2m_c2_fs$FS.err
  EPG_FIN_SPLIT=$FS timeout 900 python tools/c3_step.py > gpurun_out/r2m_c3_fs$FS.json 2> gpurun_out/r2m_c3_fs$FS.err
done
for FS in 1 0; do
  EPG_FIN_SPLIT=$FS timeout 900 ncu --set full --clock-control none -k regex:'^k_finalise_rec' -c 1 -o gpurun_out/fin_fs$FS \
      python tools/ncu_variants.py --config c2 --reps 1 --variants rb > /dev/null 2>&1
  ncu -i gpurun_out/fin_fs$FS.ncu-rep --page details > gpurun_out/r2m_fin_c2_fs$FS.txt 2>&1
  rm -f gpurun_out/fin_fs$FS.ncu-rep
done
timeout 600 python -m pytest tests/test_gpu_adaptive.py -q -x > gpurun_out/r2m_adaptive.log 2>&1
