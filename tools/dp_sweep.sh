#!/bin/bash
# DP bucket-size sweep at N GPUs (run under gpurun --gpus N)
N=${1:-2}
for K in ${BUCKETS:-8 32 128}; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29500 \
     bench.py --gpus $N --steps 20 --warmup 3 --bucket-pages $K 2>/dev/null | grep metric > gpurun_out/dp_n${N}_k${K}.json
done
