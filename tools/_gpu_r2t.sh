#!/bin/bash
# round-2 evidence for the current build: full GPU tests, smoke, default bench (C2 + C3 sub-record,
# comparators, CPU baseline), reference arm, C4 bench, ncu launch list / variants / full captures
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2t_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2t_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r2t_bench_ref.json 2> gpurun_out/r2t_bench_ref.err
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2t_bench_c4.json 2> gpurun_out/r2t_bench_c4.err
bash tools/_gpu_r2k.sh
