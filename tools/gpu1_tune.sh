#!/bin/bash
# Tuning probes: adam thread variants, K3, pack batching, lock-free speedup, actors tests.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_actors.py tests/test_gpu_lockfree.py -q > gpurun_out/pytest_actors.log 2>&1
for T in 256 512; do
  timeout 300 python bench.py --steps 50 --warmup 5 --adam-threads $T --e2e-steps 0 --no-cpu-baseline > gpurun_out/tune_adam_$T.log 2>&1
done
timeout 300 python tools/pack_bench.py --config c4 > gpurun_out/pack_c4b.log 2>&1
timeout 900 python tools/lockfree_bench.py --layers 8 --dim 8192 --batch 8192 --iters 10 > gpurun_out/lockfree_host.log 2>&1
