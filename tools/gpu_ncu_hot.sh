#!/bin/bash
# ncu --set full capture (with source) of the hot-path kernels on the C4 cone layout; the CSV pages are exported on
# the box (the .ncu-rep is dropped when it would not fit gpurun's 64 MiB return limit).
#   bash tools/gpu_ncu_hot.sh <tag> [kernel-regex] [launch-count]
set -u
TAG=${1:-ncu}
RE=${2:-'cone_kernel|k_resid|k_mu_aff|k_update_iterate'}
CNT=${3:-16}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nproc > $OUT/host.txt; free -g >> $OUT/host.txt; lscpu | head -20 >> $OUT/host.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RE" -c $CNT \
    -o $OUT/hot_kernels -f python tests/gpu_microbench.py 10000 20 250 0 1 > $OUT/ncu_full.log 2>&1
ncu -i $OUT/hot_kernels.ncu-rep --page raw --csv > $OUT/hot_kernels_raw.csv 2>/dev/null
ncu -i $OUT/hot_kernels.ncu-rep --page source --csv 2>/dev/null | gzip > $OUT/hot_kernels_source.csv.gz
ncu -i $OUT/hot_kernels.ncu-rep --page details --csv 2>/dev/null | gzip > $OUT/hot_kernels_details.csv.gz
sz=$(stat -c %s $OUT/hot_kernels.ncu-rep); if [ "$sz" -gt 40000000 ]; then rm $OUT/hot_kernels.ncu-rep; fi
tail -3 $OUT/ncu_full.log; ls -la $OUT
