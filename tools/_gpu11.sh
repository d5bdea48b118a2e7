python -m pytest tests/test_gpu_parity.py tests/test_gpu_rb.py -x -q 2>&1 | tail -3 > gpurun_out/t_par.log
python tools/c3_step.py --order growth > gpurun_out/c3_growth.json 2> gpurun_out/c3_growth.err
python tools/c3_step.py --order id > gpurun_out/c3_id.json 2> gpurun_out/c3_id.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators > gpurun_out/bench_growth.json 2> gpurun_out/bench_growth.err
timeout 900 python bench.py --no-c3 --no-cpu-baseline --no-comparators --order id > gpurun_out/bench_id.json 2> gpurun_out/bench_id.err
