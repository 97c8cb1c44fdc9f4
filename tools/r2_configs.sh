#!/bin/bash
# Round-2 single-GPU lines for the other BASELINE configs (C1, C4, C5 at 1/4/64
# MiB pages) and one ncu --set full capture of the page-Adam main kernel of
# the default (C2) bench command.  Outputs in gpurun_out/r2c_*.
cd "$(dirname "$0")/.."
run() { local name=$1; shift; timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 \
          --three-call-steps 2 "$@" > gpurun_out/r2c_$name.json 2> gpurun_out/r2c_$name.err; echo "$name rc=$?"; }
run c1 --config c1
run c4 --config c4
run c5_1m --config c5 --page-mib 1
run c5_4m --config c5
run c5_64m --config c5 --page-mib 64
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --three-call-steps 0 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/r2c_ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adam_main -s 3 -c 1 \
  -o gpurun_out/r2c_adam $CMD > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?"
