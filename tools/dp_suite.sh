#!/bin/bash
# Multi-GPU evidence for one gpurun call: probe, DP parity tests, DP bench per mode.
N=${1:-2}
mkdir -p gpurun_out
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29501 tools/symm_probe.py > gpurun_out/symm_probe_n$N.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dp.py -q > gpurun_out/pytest_dp_n$N.log 2>&1
for MODE in ${MODES:-nccl p2p nvls}; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29502 \
     bench.py --gpus $N --steps 20 --warmup 3 --dp-mode $MODE > gpurun_out/dp_n${N}_${MODE}.log 2>&1
done
# reduced-gradient deviation of the NVLS in-switch reduction vs the f32-sum oracle
DP_MODE=nvls DP_BUCKET=2 DP_DTYPE=bf16 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
   --master-addr 127.0.0.1 --master-port 29504 tests/dp_worker.py > gpurun_out/dp_worker_nvls_n$N.log 2>&1
