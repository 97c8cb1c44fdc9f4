#!/bin/bash
# Layer-group pipelined fused DP step at N=4, then 1-GPU TMA variant + reference arm.
mkdir -p gpurun_out
for MODE in p2p nvls; do
  for G in 2 4 8 16; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29505 \
       bench.py --gpus 4 --steps 20 --warmup 3 --dp-mode $MODE --dp-groups $G > gpurun_out/dppipe_n4_${MODE}_g$G.log 2>&1
  done
done
export CUDA_VISIBLE_DEVICES=0
for V in 0 1; do
  timeout 300 python bench.py --adam-variant $V --no-cpu-baseline --e2e-steps 2 > gpurun_out/c19_variant$V.log 2>&1
done
timeout 600 python bench.py --impl reference > gpurun_out/c19_ref.log 2>&1
