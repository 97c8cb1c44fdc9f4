#!/bin/bash
# Round-2 bench lines on a 2-GPU box: N=1 default, reference arm, N=2 DP (C2),
# C3 host tier DP at N=2 (8-layer slice).  Outputs in gpurun_out/r2_*.
cd "$(dirname "$0")/.."
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_n1.json 2> gpurun_out/r2_n1.err; echo "n1 rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"
python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_n2.json 2> gpurun_out/r2_n2.err; echo "n2 rc=$?"
python bench.py --gpus 2 --config c3 --c3-layers 8 --steps 3 --warmup 3 > gpurun_out/r2_c3_n2.json 2> gpurun_out/r2_c3_n2.err; echo "c3n2 rc=$?"
