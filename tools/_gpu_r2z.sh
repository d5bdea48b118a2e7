#!/bin/bash
# fused peer push (EPG_EXCHANGE=p2p): sharded tests in both modes, full GPU suite, sanitizer
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded_lib.py -q > gpurun_out/r2z_sharded.log 2>&1
echo "rc=$?" >> gpurun_out/r2z_sharded.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2z_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2z_tests.log
EPG_EXCHANGE=p2p timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py sharded > gpurun_out/r2z_san_memcheck_sharded_p2p.log 2>&1
EPG_EXCHANGE=p2p timeout 900 compute-sanitizer --tool racecheck python tools/sanitize.py sharded > gpurun_out/r2z_san_racecheck_sharded_p2p.log 2>&1
timeout 900 python tools/c3_step.py > gpurun_out/r2z_c3.json 2> gpurun_out/r2z_c3.err
