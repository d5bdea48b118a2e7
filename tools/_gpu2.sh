set -x
python -m pytest tests/test_gpu_rb.py -x -q 2>&1 | tail -15 > gpurun_out/t_rb.log
python tools/partition_bench.py c2 --leaf-parts 16 64 256 --epg2 > gpurun_out/pb_c2.json 2> gpurun_out/pb_c2.err
python tools/partition_bench.py c3 --leaf-parts 256 512 128 > gpurun_out/pb_c3.json 2> gpurun_out/pb_c3.err
python -m pytest tests/test_gpu_production.py tests/test_gpu_adaptive.py tests/test_gpu_launch_paths.py -x -q 2>&1 | tail -15 > gpurun_out/t_prod.log
python tools/partition_bench.py c4 --leaf-parts 256 > gpurun_out/pb_c4.json 2> gpurun_out/pb_c4.err
