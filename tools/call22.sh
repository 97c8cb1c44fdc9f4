#!/bin/bash
# N=2: DP tests, NVLink probe (+ncu counters), pipelined step with a persistent reduce grid.
mkdir -p gpurun_out
N=${NGPU:-2}
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x > gpurun_out/c22_pytest_dp.log 2>&1
NGPU=$N ./tools/call21.sh
for CFG in "1 0" "2 32" "2 64" "4 32" "4 64" "8 48"; do
  set -- $CFG
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus $N --steps 20 --warmup 3 --dp-mode p2p --dp-groups $1 --dp-reduce-ctas $2 --e2e-steps 0 \
     > gpurun_out/c22_n${N}_g$1_c$2.log 2>&1
done
