timeout 1200 python bench.py --config c4 --steps 20 --warmup 3 --no-comparators --no-cpu-baseline --hub-l2 1 > gpurun_out/bench_c4_l2on.json 2> gpurun_out/bench_c4_l2on.err
timeout 1200 python bench.py --config c4 --steps 20 --warmup 3 --no-comparators --no-cpu-baseline --hub-l2 0 > gpurun_out/bench_c4_l2off.json 2> gpurun_out/bench_c4_l2off.err
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
