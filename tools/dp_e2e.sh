#!/bin/bash
# DP e2e: host gradient streamed per layer group into the pipelined fused step.
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests/test_gpu_dp.py -q -k "p2p" > gpurun_out/e2e_pytest_dp_n2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29505 \
   bench.py --gpus 4 --steps 20 --warmup 3 > gpurun_out/e2e_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
   bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/e2e_n2.log 2>&1
