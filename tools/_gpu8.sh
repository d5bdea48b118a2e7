python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_hubs.py tests/test_gpu_launch_paths.py tests/test_gpu_sharded_lib.py tests/test_gpu_run_host.py -x -q 2>&1 | tail -3 > gpurun_out/t_par.log
python tools/c3_step.py > gpurun_out/c3_step.json 2> gpurun_out/c3_step.err
