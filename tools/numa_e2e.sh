#!/bin/bash
# e2e with / without binding each rank to its GPU's NUMA node (N=4, N=1).
mkdir -p gpurun_out
for f in /sys/devices/system/node/node*/cpulist; do echo "$f $(cat $f)"; done > gpurun_out/numa_topo.txt
nvidia-smi topo -m >> gpurun_out/numa_topo.txt 2>&1
for B in 0 1; do
  if [ $B = 1 ]; then export HM_NO_NUMA_BIND=1; else unset HM_NO_NUMA_BIND; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/numa_n4_nobind$B.log 2>&1
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/numa_n1_nobind$B.log 2>&1
done
