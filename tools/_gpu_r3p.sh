#!/bin/bash
# the multi-GPU bench path through a one-rank NCCL communicator (C3 via epg_run_sharded), both exchanges
mkdir -p gpurun_out
timeout 1200 python bench.py --force-sharded --steps 10 --warmup 3 > gpurun_out/r3p_sharded.json 2> gpurun_out/r3p_sharded.err
echo "rc=$?" >> gpurun_out/r3p_sharded.err
timeout 1200 python bench.py --force-sharded --exchange p2p --steps 10 --warmup 3 > gpurun_out/r3p_sharded_p2p.json 2> gpurun_out/r3p_sharded_p2p.err
echo "rc=$?" >> gpurun_out/r3p_sharded_p2p.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r3p_torchrun.json 2> gpurun_out/r3p_torchrun.err
echo "rc=$?" >> gpurun_out/r3p_torchrun.err
