#!/usr/bin/env python
"""Turn one gpurun_out/<tag>/ directory (written by tools/gpu_round.sh) into the tracked summaries under profiles/:

    profiles/<tag>_launches_by_kernel.csv   per-kernel count / total device time / share of the ncu launch list
    profiles/<tag>_launches.csv.gz          the launch list itself (gpu__time_duration.sum per launch)
    profiles/<tag>_hot_kernels_ncu.csv      selected `ncu --set full` metrics of the hot-path kernels, per launch
    profiles/<tag>_bench.json, _bench_reference.json, _microbench.txt, _pytest_gpu.log, _smoke.log
    profiles/dominant_kernel_traffic.json   dram bytes per launch of the dominant kernel (read by bench.py)

usage: python tools/summarize_profiles.py r01a [kernel-regex-of-the-dominant-kernel]
"""
import collections
import csv
import gzip
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
dominant = sys.argv[2] if len(sys.argv) > 2 else r"k_neg_wtw<2, 1"
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles")
os.makedirs(dst, exist_ok=True)

for name in ("bench.json", "bench_reference.json", "microbench.txt", "pytest_gpu.log", "smoke.log", "gpu.txt",
             "bench_torchrun1.json", "bench_C1_random_qp.json", "bench_C2_lasso.json", "bench_C3_portfolio.json",
             "bench_C5_mpc.json", "bench_C2_lasso_20k.json", "bench_C4_group_lasso_survey.json", "c5_batch_throughput.txt", "c5_batched_throughput.txt",
             "ldl_factor_solve_ms.txt"):
    p = os.path.join(src, name)
    if os.path.exists(p) and os.path.getsize(p) > 0:
        shutil.copy(p, os.path.join(dst, f"{tag}_{name}"))

lp = os.path.join(src, "launches.csv")
if not os.path.exists(lp) and os.path.exists(lp + ".gz"):  # the round script compresses it on the box
    with gzip.open(lp + ".gz", "rt") as f, open(lp, "w") as g:
        g.write(f.read())
if os.path.exists(lp):
    lines = [ln for ln in open(lp) if ln.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for row in rd:
        name = re.sub(r"\(.*", "", row[ki]).replace("<unnamed>::", "").replace("void ", "")
        v = float(row[vi].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(row[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    with open(os.path.join(dst, f"{tag}_launches_by_kernel.csv"), "w") as f:
        f.write("kernel,launches,total_us,mean_us,share\n")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"\"{k}\",{cnt[k]},{v:.1f},{v / cnt[k]:.2f},{v / T:.4f}\n")
    with gzip.open(os.path.join(dst, f"{tag}_launches.csv.gz"), "wt") as f:
        f.writelines(lines)

rep = os.path.join(src, "hot_kernels.ncu-rep")
rawcsv = os.path.join(src, "hot_kernels_raw.csv")  # exported on the box when the report is too large to travel
if os.path.exists(rep) or os.path.exists(rawcsv):
    raw = (open(rawcsv).read() if os.path.exists(rawcsv) else
           subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "smsp__issue_active.avg.pct_of_peak_sustained_active"]
    idx = [hdr.index(w) for w in want if w in hdr]
    traffic = {}
    with open(os.path.join(dst, f"{tag}_hot_kernels_ncu.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow([f"{hdr[i]} [{units[i]}]" if units[i] else hdr[i] for i in idx])
        for row in rows[2:]:
            row = list(row)
            row[hdr.index("Kernel Name")] = re.sub(r"\(.*", "", row[hdr.index("Kernel Name")]).replace("<unnamed>::", "")
            w.writerow([row[i] for i in idx])
            if re.search(dominant, row[hdr.index("Kernel Name")]):
                def tobytes(col):
                    v = float(row[hdr.index(col)].replace(",", ""))
                    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[hdr.index(col)]]
                traffic.setdefault("samples", []).append(tobytes("dram__bytes_read.sum") + tobytes("dram__bytes_write.sum"))
    if traffic.get("samples"):
        tp = os.path.join(dst, "dominant_kernel_traffic.json")
        cur = json.load(open(tp)) if os.path.exists(tp) else {}
        cur["C4_group_lasso"] = sum(traffic["samples"]) / len(traffic["samples"])
        cur["source"] = f"profiles/{tag}_hot_kernels_ncu.csv ({dominant}, mean of {len(traffic['samples'])} launches, C4 cone layout)"
        json.dump(cur, open(tp, "w"), indent=1)
for extra in ("hot_kernels_source.csv.gz",):
    p = os.path.join(src, extra)
    if os.path.exists(p):
        shutil.copy(p, os.path.join(dst, f"{tag}_{extra}"))
print("profiles/ updated from", src)
