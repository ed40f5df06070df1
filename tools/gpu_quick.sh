#!/bin/bash
# Quick GPU check between changes: parity tests + kernel microbenchmark (+ optional short bench).
#   bash tools/gpu_quick.sh <tag> [bench]
set -u
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
tail -15 $OUT/pytest_gpu.log
python tests/gpu_microbench.py > $OUT/microbench.txt 2>&1; head -20 $OUT/microbench.txt
if [ "${2:-}" = "bench" ]; then
  python bench.py --steps 2 --warmup 1 --e2e-steps 1 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
  cut -c1-1800 $OUT/bench.json; tail -5 $OUT/bench.err
fi
