#!/bin/bash
# DP step on the other BASELINE configs (C1 GPT-2 124M, C4 T5-MoE small pages) at N=2 and N=4.
mkdir -p gpurun_out
for CFG in c1 c4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 4 --config $CFG --steps 20 --warmup 3 --e2e-steps 2 > gpurun_out/dpc_${CFG}_n4.log 2>&1
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port 29506 bench.py --gpus 2 --config $CFG --steps 20 --warmup 3 --e2e-steps 2 > gpurun_out/dpc_${CFG}_n2.log 2>&1
done
