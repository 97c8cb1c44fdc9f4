#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dp.py -q > gpurun_out/w3_pytest_n2.log 2>&1
for W in 1 0; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 2 --steps 30 --warmup 3 --dp-reduce-wide $W --e2e-steps 0 > gpurun_out/w3_n2_w$W.log 2>&1
done
for C in 96 160; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 2 --steps 30 --warmup 3 --dp-groups 8 --dp-reduce-ctas $C --e2e-steps 0 > gpurun_out/w3_n2_c$C.log 2>&1
done
