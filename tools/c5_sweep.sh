#!/bin/bash
# C5: GPT-3 175B single-layer slice, page size 1..64 MiB (N=1 sweep; N>1 DP step with MODE)
N=${1:-1}
mkdir -p gpurun_out
for P in ${PAGES:-1 2 4 8 16 32 64}; do
  if [ "$N" = "1" ]; then
    timeout 300 python bench.py --config c5 --page-mib $P --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/c5_n1_p$P.log 2>&1
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29503 \
      bench.py --gpus $N --config c5 --page-mib $P --steps 10 --warmup 3 --dp-mode ${MODE:-p2p} --bucket-pages 4 --e2e-steps 0 \
      > gpurun_out/c5_n${N}_p$P.log 2>&1
  fi
done
