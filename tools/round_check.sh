#!/bin/bash
# What the driver runs at round end, on one box: GPU tests, smoke, default bench
# lines (N=1, reference arm, N=2, N=4 when the box has the GPUs).
# SKIP_TESTS=1: bench lines only.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
if [ -z "$SKIP_TESTS" ]; then
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/rc_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_pytest_gpu.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rc_smoke.log 2>&1
fi
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/rc_bench_n1.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/rc_bench_ref.log 2>&1
for N in 2 4 8; do
  [ $NG -ge $N ] || continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 29507 bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/rc_bench_n$N.log 2>&1
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port 29508 bench.py --impl reference --gpus $N --steps 20 --warmup 5 > gpurun_out/rc_bench_ref_n$N.log 2>&1
done
