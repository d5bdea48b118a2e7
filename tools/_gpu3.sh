python -m pytest tests/test_gpu_rb.py -x -q 2>&1 | tail -5 > gpurun_out/t_rb.log
EPG_RB_TRACE=1 python tools/partition_bench.py c3 --leaf-parts 512 > gpurun_out/pb_c3.json 2> gpurun_out/pb_c3.err
EPG_RB_TRACE=1 python tools/partition_bench.py c4 --leaf-parts 512 4096 > gpurun_out/pb_c4.json 2> gpurun_out/pb_c4.err
