#!/bin/bash
# ncu --set full of the fused DP kernels (GPU 0 alone, peers mapped), N=2.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on --devices 0 \
  -k regex:"reduce_check|adam_main" -c 2 -o gpurun_out/dp_full \
  python tools/nvlink_probe.py --gpus 2 --reps 1 --solo > gpurun_out/dp_full.log 2>&1
ncu -i gpurun_out/dp_full.ncu-rep --page raw --csv > gpurun_out/dp_full_raw.csv 2>/dev/null
