#!/bin/bash
# Fused DP step: modes x layer-group pipelining at N GPUs.
N=${1:-4}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dp.py -q > gpurun_out/pytest_dp_pipe_n$N.log 2>&1
for MODE in p2p nvls; do
  for G in ${GROUPS_LIST:-1 4 8}; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29505 \
       bench.py --gpus $N --steps 20 --warmup 3 --dp-mode $MODE --dp-groups $G > gpurun_out/dppipe_n${N}_${MODE}_g$G.log 2>&1
  done
done
