#!/bin/bash
# Bulk-copy all-gather epilogue (hm_set_ag_publish): parity (DP tests), timing, ncu HBM/NVLink bytes.
mkdir -p gpurun_out
N=${NGPU:-2}
timeout 900 python -m pytest tests/test_gpu_dp.py -q -x -k "bulk or p2p" > gpurun_out/agp_pytest_n$N.log 2>&1
timeout 600 python tools/nvlink_probe.py --gpus $N --reps 3 --ag-publish 0 1 2 > gpurun_out/agp_probe_n$N.log 2>&1
timeout 900 ncu --devices 0 -k regex:"adam_main" -c 6 --clock-control none \
  --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum \
  --csv --log-file gpurun_out/agp_ncu_n$N.csv python tools/nvlink_probe.py --gpus $N --reps 1 --solo --ag-publish 1 2 > gpurun_out/agp_ncu_n$N.log 2>&1
for P in 0 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29505 \
     bench.py --gpus $N --steps 20 --warmup 3 --ag-publish $P --e2e-steps 0 > gpurun_out/agp_bench_n${N}_p$P.log 2>&1
done
