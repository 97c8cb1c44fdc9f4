#!/bin/bash
# NVLS layer-group pipeline (outbound-heavy multimem reduce of group k+1 beside
# the inbound-heavy multimem all-gather of group k) vs the P2P step, C2.
cd "$(dirname "$0")/.."
N=${N:-4}
run() { local name=$1; shift; timeout 300 python bench.py --gpus $N --steps 20 --warmup 5 --e2e-steps 0 "$@" \
          > gpurun_out/nv_$name.json 2> gpurun_out/nv_$name.err; echo "$name rc=$?"; }
run p2p
run nvls --dp-mode nvls --dp-groups 1
run nvls_g8_c128 --dp-mode nvls --dp-groups 8 --dp-reduce-ctas 128
run nvls_g8_c256 --dp-mode nvls --dp-groups 8 --dp-reduce-ctas 256
run nvls_g16_c128 --dp-mode nvls --dp-groups 16 --dp-reduce-ctas 128
run nvls_g4_c64 --dp-mode nvls --dp-groups 4 --dp-reduce-ctas 64
run nvls_g8_c128_u512 --dp-mode nvls --dp-groups 8 --dp-reduce-ctas 128 --dp-update-ctas 512
