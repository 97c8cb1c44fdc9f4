#!/bin/bash
# Round-2 DP lines for BASELINE config 5 (GPT-3 175B layer slice, page size
# 1 / 4 / 64 MiB) at N = 2 and 4 with the round-2 default policy (N=2: the
# one-pass kernel; N=4: the two-phase fused P2P step).  Outputs in
# gpurun_out/r2dp_*.json.  Needs a 4-GPU box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in 2 4; do
  for P in 1 4 64; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 2955$N bench.py --gpus $N --config c5 --page-mib $P --bucket-pages 4 --steps 20 \
      --warmup 5 --e2e-steps 2 --no-cpu-baseline > gpurun_out/r2dp_c5_n${N}_p${P}.json \
      2> gpurun_out/r2dp_c5_n${N}_p${P}.err
    echo "c5 N=$N P=$P rc=$?"
  done
done
