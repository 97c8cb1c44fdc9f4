#!/bin/bash
# DP parity at N=4 and N=2 with the final defaults, plus default bench lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dp.py -q > gpurun_out/df_pytest_n4.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29505 \
   bench.py --gpus 4 > gpurun_out/df_n4.log 2>&1
export CUDA_VISIBLE_DEVICES=0,1
timeout 1200 python -m pytest tests/test_gpu_dp.py -q > gpurun_out/df_pytest_n2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
   bench.py --gpus 2 > gpurun_out/df_n2.log 2>&1
