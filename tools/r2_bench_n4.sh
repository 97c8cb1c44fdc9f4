#!/bin/bash
# Round-2 bench lines on a 4-GPU box: C2 DP step (p2p default, NVLS
# unpipelined and layer-group pipelined), C3 at full size on the DP-sharded
# pinned-host tier.  Outputs in gpurun_out/r2n4_*.
cd "$(dirname "$0")/.."
run() { local name=$1; shift; timeout ${T:-420} "$@" > gpurun_out/r2n4_$name.json 2> gpurun_out/r2n4_$name.err; echo "$name rc=$?"; }
run c2_p2p python bench.py --gpus 4 --steps 20 --warmup 5
run c2_nvls python bench.py --gpus 4 --steps 20 --warmup 5 --dp-mode nvls --e2e-steps 0
run c2_nvls_g8 python bench.py --gpus 4 --steps 20 --warmup 5 --dp-mode nvls --dp-groups 8 --dp-reduce-ctas 128 --e2e-steps 0
run c2_p2p_g8 python bench.py --gpus 4 --steps 20 --warmup 5 --dp-groups 8 --dp-reduce-ctas 128 --e2e-steps 0
T=1200 run c3_full python bench.py --gpus 4 --config c3 --steps 3 --warmup 3
