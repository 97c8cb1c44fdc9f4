#!/bin/bash
# N GPUs: DP tests incl. the persistent reduce grid, then pipelined step sweep over reduce grids.
mkdir -p gpurun_out
N=${NGPU:-2}
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x > gpurun_out/c24_pytest_dp_n$N.log 2>&1
for CFG in "1 0" "2 64" "2 128" "4 64" "4 128" "4 148" "8 128"; do
  set -- $CFG
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus $N --steps 20 --warmup 3 --dp-mode p2p --dp-groups $1 --dp-reduce-ctas $2 --e2e-steps 0 \
     > gpurun_out/c24_n${N}_g$1_c$2.log 2>&1
done
