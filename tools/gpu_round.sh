#!/bin/bash
# One gpurun call: GPU parity tests, the bench line, the ncu launch list of the same bench command and one
# `ncu --set full` capture of the dominant kernel.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_round.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,memory.total --format=csv > $OUT/gpu.txt 2>&1
python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/smoke.log
# the two commands the driver runs at round end, with its flags
T0=$SECONDS; python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$? wall $((SECONDS-T0)) s" | tee $OUT/bench_wall.txt
T0=$SECONDS; python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "reference arm rc=$? wall $((SECONDS-T0)) s" | tee -a $OUT/bench_wall.txt
python tests/gpu_microbench.py > $OUT/microbench.txt 2>&1
# the other BASELINE configurations (parity-size cases, not the headline) and the C5 batch on one GPU
for w in C1_random_qp C2_lasso C2_lasso_20k C3_portfolio C5_mpc C4_group_lasso_survey; do
  python bench.py --workload $w --no-batch --cpu-budget 20 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
python tests/gpu_batched_throughput.py 512 > $OUT/c5_batched_throughput.txt 2>&1
python tests/gpu_factor_profile.py > $OUT/ldl_factor_solve_ms.txt 2>&1
# the torchrun launch the driver uses for N > 1, here with one rank (NCCL init, barrier, max over ranks)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu --no-ladder > $OUT/bench_torchrun1.json 2> $OUT/bench_torchrun1.err
# launch list of the bench command (resident arm only: setup + ONE solve; shares, not absolutes)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu --no-ladder --no-batch --e2e-steps 0 > $OUT/bench_under_ncu.log 2>&1
gzip -f $OUT/launches.csv
# full capture of the dominant hot-path kernel (and the other cone kernels) on the C4 cone layout
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_neg_wtw|cone_kernel|k_resid|k_mu_aff|k_update_iterate' -c 16 \
    -o $OUT/hot_kernels -f python tests/gpu_microbench.py 10000 20 250 0 1 > $OUT/ncu_full.log 2>&1
# gpurun_out/ travels back only below 64 MiB: keep the raw-metric and source pages as CSV, drop a large report
ncu -i $OUT/hot_kernels.ncu-rep --page raw --csv > $OUT/hot_kernels_raw.csv 2> /dev/null
ncu -i $OUT/hot_kernels.ncu-rep --page source --csv 2> /dev/null | gzip > $OUT/hot_kernels_source.csv.gz
[ $(stat -c %s $OUT/hot_kernels.ncu-rep) -gt 30000000 ] && rm -f $OUT/hot_kernels.ncu-rep
ls -la $OUT
tail -3 $OUT/pytest_gpu.log; cat $OUT/bench.json | cut -c1-3000
