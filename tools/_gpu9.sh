bash tools/profile_round.sh c2 rb,ep1,default,naive > gpurun_out/prof_c2.log 2>&1
python tools/summarize_ncu.py --config c2 --round r02 > gpurun_out/sum_c2.log 2>&1
bash tools/profile_round.sh c3 rb,default,naive > gpurun_out/prof_c3.log 2>&1
python tools/summarize_ncu.py --config c3 --round r02 --m 127708987 > gpurun_out/sum_c3.log 2>&1
for c in c2 c3; do
  ncu -i gpurun_out/full_fin_$c.ncu-rep --page details > gpurun_out/full_fin_$c.txt 2>&1
  ncu -i gpurun_out/full_edge_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_edge_$c.csv 2>&1
done
mkdir -p gpurun_out/prof
cp profiles/r02_* profiles/traffic_* gpurun_out/prof/ 2>/dev/null
rm -f gpurun_out/full_fin_*.ncu-rep gpurun_out/full_edge_c2.ncu-rep
gzip -f gpurun_out/sass_edge_*.csv
ls -la gpurun_out gpurun_out/prof
