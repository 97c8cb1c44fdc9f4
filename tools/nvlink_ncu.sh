#!/bin/bash
# Single-process NVLink probe of the fused DP kernels + ncu NVLink byte counters on GPU 0.
mkdir -p gpurun_out
timeout 600 python tools/nvlink_probe.py --gpus ${NGPU:-2} --reps 5 > gpurun_out/nvprobe.log 2>&1 || exit 1
timeout 900 ncu --devices 0 -k regex:"reduce_check|adam_main" -c 2 --clock-control none \
  --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__occupancy_limit_registers \
  --csv --log-file gpurun_out/nvprobe_ncu.csv python tools/nvlink_probe.py --gpus ${NGPU:-2} --reps 1 --solo > gpurun_out/nvprobe_ncu.log 2>&1
