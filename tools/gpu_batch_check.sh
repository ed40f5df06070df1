#!/bin/bash
# Batched small-problem mode on the GPU: parity tests, then throughput of the 512-instance C5 batch by batch size.
#   bash tools/gpu_batch_check.sh <tag>
set -u
TAG=${1:-batch}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_step_vectors.py -x -q > $OUT/pytest_batched.log 2>&1; echo "pytest rc=$?"
tail -n 30 $OUT/pytest_batched.log
timeout 900 python tests/gpu_batched_throughput.py > $OUT/c5_batched_throughput.txt 2>&1; echo "throughput rc=$?"
tail -n 20 $OUT/c5_batched_throughput.txt
