#!/bin/bash
# C3 DP host tier at N=4: staging slots / page-group size sweep on an
# 8-layer slice (the per-rank PCIe fraction is size-independent).
cd "$(dirname "$0")/.."
run() { local name=$1; shift; timeout 600 python bench.py --gpus 4 --config c3 --c3-layers 8 --steps 3 --warmup 3 \
          --c3-lockfree-iters 0 "$@" > gpurun_out/c3s_$name.json 2> gpurun_out/c3s_$name.err; echo "$name rc=$?"; }
run s2_g64 --swap-slots 2 --swap-group-pages 64
run s3_g64 --swap-slots 3 --swap-group-pages 64
run s2_g32 --swap-slots 2 --swap-group-pages 32
run s3_g32 --swap-slots 3 --swap-group-pages 32
run s2_g128 --swap-slots 2 --swap-group-pages 128
