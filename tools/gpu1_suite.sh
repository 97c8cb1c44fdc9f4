#!/bin/bash
# Single-GPU evidence: GPU tests, bench C2 (default line), C1, C4, C5 sweep, C3 swap tier, C4 pack.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --e2e-steps 3 --cpu-sample-pages 16 > gpurun_out/bench_c1.log 2>&1
timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --e2e-steps 2 --cpu-sample-pages 64 > gpurun_out/bench_c4.log 2>&1
timeout 300 python tools/pack_bench.py --config c4 > gpurun_out/pack_c4.log 2>&1
PAGES="1 4 16 64" ./tools/c5_sweep.sh 1
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --c3-layers 8 > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
