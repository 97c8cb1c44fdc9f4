#!/bin/bash
# C5 page-size sweep on the DP step at N=2 and N=4.
PAGES="1 4 16 64" ./tools/c5_sweep.sh 4
CUDA_VISIBLE_DEVICES=0,1 PAGES="1 4 16 64" ./tools/c5_sweep.sh 2
