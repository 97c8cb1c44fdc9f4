#!/bin/bash
# Refresh the single-GPU config lines with the current kernels.
mkdir -p gpurun_out
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --e2e-steps 3 --cpu-sample-pages 16 > gpurun_out/cr_c1.log 2>&1
timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --e2e-steps 2 --cpu-sample-pages 64 > gpurun_out/cr_c4.log 2>&1
timeout 300 python bench.py --config c5 --page-mib 4 --steps 20 --warmup 3 --e2e-steps 2 --cpu-sample-pages 16 > gpurun_out/cr_c5.log 2>&1
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --c3-layers 8 > gpurun_out/cr_c3.log 2>&1
timeout 300 python tools/pack_bench.py --config c4 > gpurun_out/cr_pack_c4.log 2>&1
