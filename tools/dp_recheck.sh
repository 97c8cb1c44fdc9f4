#!/bin/bash
# After a DP kernel change: parity at N=4, HBM bytes of the peer-publish kernel, N=2/N=4 bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x > gpurun_out/dr_pytest_dp_n4.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/publish_probe.py > gpurun_out/dr_pubprobe.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu -k regex:adam_main -c 2 --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum \
  --csv --log-file gpurun_out/dr_pubprobe_ncu.csv python tools/publish_probe.py > /dev/null 2>&1
timeout 600 python tools/nvlink_probe.py --gpus 4 --reps 5 > gpurun_out/dr_probe_n4.log 2>&1
run() {  # N G CTAS tag
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus $1 --steps 20 --warmup 3 --dp-groups $2 --dp-reduce-ctas $3 --e2e-steps 0 > gpurun_out/dr_n$1_g$2_c$3.log 2>&1
}
run 4 1 0; run 4 4 128
export CUDA_VISIBLE_DEVICES=0,1
timeout 600 python tools/nvlink_probe.py --gpus 2 --reps 5 > gpurun_out/dr_probe_n2.log 2>&1
run 2 1 0; run 2 8 128; run 2 4 128
