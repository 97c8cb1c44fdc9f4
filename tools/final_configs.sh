#!/bin/bash
# Final-code lines for every BASELINE config on one B200 (C1, C2, C4, C5 page sweep, C3 host + SSD tiers).
mkdir -p gpurun_out
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --e2e-steps 3 --cpu-sample-pages 16 > gpurun_out/fc_c1.log 2>&1
timeout 300 python bench.py --config c2 > gpurun_out/fc_c2.log 2>&1
timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --e2e-steps 2 --cpu-sample-pages 64 > gpurun_out/fc_c4.log 2>&1
for P in 1 4 16 64; do
  timeout 300 python bench.py --config c5 --page-mib $P --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/fc_c5_p$P.log 2>&1
done
timeout 900 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/fc_c3_host.log 2>&1
timeout 1200 python bench.py --config c3 --state-tier ssd --c3-layers 2 --steps 2 --warmup 3 > gpurun_out/fc_c3_ssd.log 2>&1
