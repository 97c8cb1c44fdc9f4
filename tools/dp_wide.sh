#!/bin/bash
# 256-bit peer loads in the fused reduce: parity, probe timing (N=4), ncu NVLink bytes, full step.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -k "ld256 or wide8" > gpurun_out/wd_pytest.log 2>&1
timeout 600 python tools/nvlink_probe.py --gpus 4 --reps 5 > gpurun_out/wd_probe_n4.log 2>&1
for W in 0 1; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 4 --steps 30 --warmup 3 --dp-reduce-wide $W --e2e-steps 0 > gpurun_out/wd_n4_w$W.log 2>&1
done
