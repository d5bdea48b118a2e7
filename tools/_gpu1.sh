set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -i "model name"
python tools/flush_floor.py > gpurun_out/flush_floor.json 2> gpurun_out/flush_floor.err
for t in memcheck racecheck synccheck; do
  for s in c1_single c1_multiwave default_map hub spmv; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py $s > gpurun_out/san_${t}_${s}.log 2>&1
    echo "$t $s rc=$?" >> gpurun_out/san_summary.txt
  done
done
