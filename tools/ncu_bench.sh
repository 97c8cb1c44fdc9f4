#!/bin/bash
# ncu evidence of the default bench command itself (after it exits 0 without ncu):
# launch list (cold-cache, serialised) and one --set full capture each of the
# page-Adam main kernel and the K3 accumulate kernel (first-message form).
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --three-call-steps 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/nb_plain.log 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
  --log-file gpurun_out/nb_launches.csv $CMD > gpurun_out/nb_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"adam_main|accumulate_kernel" -s 8 -c 2 \
  -o gpurun_out/nb_full $CMD > gpurun_out/nb_full.log 2>&1
