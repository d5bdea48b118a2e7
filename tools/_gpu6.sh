python -m pytest tests/test_gpu_sharded_lib.py tests/test_gpu_shard.py -x -q 2>&1 | tail -8 > gpurun_out/t_sh.log
timeout 900 python bench.py --force-sharded --config c3 --steps 10 --warmup 3 > gpurun_out/bench_sh_c3.json 2> gpurun_out/bench_sh_c3.err
