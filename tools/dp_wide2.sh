#!/bin/bash
# 256-bit reduce: ncu NVLink bytes (GPU 0 alone, N=4 peers) and the N=2 steps.
mkdir -p gpurun_out
timeout 900 ncu --devices 0 -k regex:reduce_check -c 2 --clock-control none \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum \
  --csv --log-file gpurun_out/wd_ncu.csv python tools/nvlink_probe.py --gpus 4 --reps 1 --solo > gpurun_out/wd_ncu.log 2>&1
export CUDA_VISIBLE_DEVICES=0,1
for CFG in "1 0 0" "1 0 1" "8 128 0"; do
  set -- $CFG
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 2 --steps 30 --warmup 3 --dp-groups $1 --dp-reduce-ctas $2 --dp-reduce-wide $3 --e2e-steps 0 \
     > gpurun_out/wd_n2_g$1_w$3.log 2>&1
done
