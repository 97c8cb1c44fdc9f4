#!/bin/bash
# Pipelined DP step with a persistent reduce grid: N=4 and more N=2 points.
mkdir -p gpurun_out
run() {  # N G CTAS
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus $1 --steps 20 --warmup 3 --dp-mode p2p --dp-groups $2 --dp-reduce-ctas $3 --e2e-steps 0 \
     > gpurun_out/c25_n$1_g$2_c$3.log 2>&1
}
run 4 1 0; run 4 4 128; run 4 8 128; run 4 8 192; run 4 16 148
export CUDA_VISIBLE_DEVICES=0,1
run 2 8 192; run 2 8 256; run 2 16 128; run 2 16 192; run 2 8 96
