#!/bin/bash
# N=2: layer-group pipelining of the fused DP step (RS link-bound, update HBM-bound) + DP e2e leg.
mkdir -p gpurun_out
for G in 1 2 4 8; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 2 --steps 20 --warmup 3 --dp-mode p2p --dp-groups $G > gpurun_out/dppipe_n2_p2p_g$G.log 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
   bench.py --gpus 2 --steps 20 --warmup 3 --dp-mode nccl > gpurun_out/dppipe_n2_nccl.log 2>&1
