#!/bin/bash
# N=2 pipelined DP step with the reduce and the update in two green contexts.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -k "green or ingest" > gpurun_out/gr_pytest.log 2>&1
run() {  # G SMS
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 2 --steps 20 --warmup 3 --dp-groups $1 --dp-reduce-sms $2 --dp-reduce-ctas 0 --e2e-steps 0 \
     > gpurun_out/gr_g$1_s$2.log 2>&1
}
run 8 16; run 8 24; run 8 32; run 8 48; run 4 32; run 16 32; run 8 64
