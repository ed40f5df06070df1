#!/bin/bash
# ncu --set full capture (with source) of the hot-path kernels on the C4 cone layout.
#   bash tools/gpu_ncu_hot.sh <tag> [kernel-regex] [launch-count]
set -u
TAG=${1:-ncu}
RE=${2:-'k_neg_wtw|cone_kernel|k_resid|k_mu_aff|k_update_iterate'}
CNT=${3:-40}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nproc > $OUT/host.txt; free -g >> $OUT/host.txt; lscpu | head -20 >> $OUT/host.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RE" -c $CNT \
    -o $OUT/hot_kernels -f python tests/gpu_microbench.py 10000 20 250 0 1 > $OUT/ncu_full.log 2>&1
tail -3 $OUT/ncu_full.log; ls -la $OUT
