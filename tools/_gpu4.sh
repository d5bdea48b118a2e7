python -m pytest tests/test_gpu_rb.py -x -q 2>&1 | tail -3 > gpurun_out/t_rb.log
EPG_RB_TRACE=1 timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
