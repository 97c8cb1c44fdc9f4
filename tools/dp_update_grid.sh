#!/bin/bash
# N=2 pipelined DP step: persistent update grid sweep (plus parity of that path).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -k "p2p" > gpurun_out/ug_pytest_dp_n2.log 2>&1
run() {  # G C U
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 2 --steps 20 --warmup 3 --dp-groups $1 --dp-reduce-ctas $2 --dp-update-ctas $3 --e2e-steps 0 \
     > gpurun_out/ug_g$1_c$2_u$3.log 2>&1
}
run 8 128 0; run 8 128 148; run 8 128 222; run 8 128 296; run 8 128 370; run 8 64 296; run 8 96 222; run 4 128 296; run 16 128 296
