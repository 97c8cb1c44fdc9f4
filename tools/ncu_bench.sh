#!/bin/bash
# ncu evidence of the default bench command itself (after it exits 0 without ncu):
# launch list (cold-cache, serialised) and one --set full capture of adam_main.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/nb_plain.log 2>&1 || exit 1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/nb_launches.csv $CMD > gpurun_out/nb_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:adam_main -s 5 -c 1 \
  -o gpurun_out/nb_full $CMD > gpurun_out/nb_full.log 2>&1
