#!/bin/bash
# hub / peer reductions as explicit RED (the peer push's system fence had turned the hub split's
# reductions into returning ATOMGs): GPU suite, C4 A/B, C2 + C3, p2p sanitizer
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r3k_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3k_tests.log
EPG_EXCHANGE=p2p timeout 600 python -m pytest tests/test_gpu_sharded_lib.py -q > gpurun_out/r3k_p2p.log 2>&1
echo "rc=$?" >> gpurun_out/r3k_p2p.log
EPG_EXCHANGE=p2p timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py sharded > gpurun_out/r3k_san_memcheck_p2p.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py hub > gpurun_out/r3k_san_memcheck_hubs.log 2>&1
timeout 900 python bench.py --config c4 --no-cpu-baseline --no-comparators > gpurun_out/r3k_c4_new.json 2> gpurun_out/r3k_c4_new.err
timeout 900 python bench.py --no-cpu-baseline --no-comparators > gpurun_out/r3k_c2_new.json 2> gpurun_out/r3k_c2_new.err
