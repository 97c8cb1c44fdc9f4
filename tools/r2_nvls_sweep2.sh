#!/bin/bash
# NVLS layer-group pipeline, second sweep: SM partition by green contexts vs
# persistent grids (C2, N=4).
cd "$(dirname "$0")/.."
N=${N:-4}
run() { local name=$1; shift; timeout 300 python bench.py --gpus $N --steps 20 --warmup 5 --e2e-steps 0 --dp-mode nvls "$@" \
          > gpurun_out/nv2_$name.json 2> gpurun_out/nv2_$name.err; echo "$name rc=$?"; }
run g8_sms24 --dp-groups 8 --dp-reduce-sms 24
run g8_sms40 --dp-groups 8 --dp-reduce-sms 40
run g8_sms56 --dp-groups 8 --dp-reduce-sms 56
run g8_c64 --dp-groups 8 --dp-reduce-ctas 64
run g8_c128_u256 --dp-groups 8 --dp-reduce-ctas 128 --dp-update-ctas 256
run g8_c128_u1024 --dp-groups 8 --dp-reduce-ctas 128 --dp-update-ctas 1024
run g12_c128_u512 --dp-groups 12 --dp-reduce-ctas 128 --dp-update-ctas 512
