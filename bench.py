#!/usr/bin/env python
"""Benchmark of the IPM hot path (BASELINE.json: "IPM solve time (s); cone+KKT-update
us/iter vs HBM roofline; speedup vs CPU").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload NAME]

A step is ONE complete interior-point solve of the workload (initial point +
every iteration until the reference's termination test passes).  Workload at
N=1: C4, the ~1.2e8-KKT-nonzero group-lasso SOCP (10^4 second-order cones of
size 20..250) -- the configuration BASELINE.json's target is quoted on.

  value  seconds per solve with the problem, KKT system and factor analysis
         already resident in HBM when the timed region starts (CUDA events);
  e2e    seconds per Solver(algebra="cuda").setup(...).solve() call starting
         from HOST NumPy buffers: KKT assembly, ordering, H2D, solve, D2H;
  roofline   the dominant hot-path kernel (the -W'W generate-and-scatter):
         algorithmic bytes / CUDA-event time vs the measured HBM peak;
  cpu_baseline  the CPU oracle (C port of the reference) on a bounded sample.

N > 1 (torchrun): every rank solves its own independent instance (seed = rank):
no data-path collective, weak scaling, value = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name -> (config key, kwargs, CPU sample kwargs, scale = full work / sample work)
    "C4_group_lasso": ("C4_group_lasso", dict(groups=10_000, qlo=20, qhi=250, samples=2_000, nnz_per_col=3),
                       dict(groups=16, qlo=20, qhi=250, samples=2_000, nnz_per_col=3)),
    "C2_lasso": ("C2_lasso", dict(features=100_000, samples=5_000), dict(features=2_000, samples=100)),
    "C3_portfolio": ("C3_portfolio", dict(assets=100_000, factors=100, sector=100),
                     dict(assets=2_000, factors=100, sector=100)),
    "C1_random_qp": ("C1_random_qp", dict(n=2000, p=500, m=4000), dict(n=1000, p=250, m=2000)),
    "C5_mpc": ("C5_mpc", dict(horizon=50, nx=12, nu=4), dict(horizon=50, nx=12, nu=4)),
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return float(json.load(open(path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = [ln.strip().split(", ") for ln in open(self.f.name) if ln.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[k] for r in rows if len(r) >= 7 for k in range(4) if r[3 + k].strip() == "Active"})
        pw = [float(r[2]) for r in rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(rows), "reasons": reasons}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ------------------------------------------------------------------ CPU arms
def cpu_solve_sample(workload, threads_note=True):
    """One oracle solve of the bounded CPU sample; returns (seconds_setup, seconds_solve, iterations, scale, text)."""
    from oracle import qsocp_oracle as orc
    from paper_2603_29197_b200 import configs

    key, full_kw, sample_kw = WORKLOADS[workload]
    d = configs.make(key, **sample_kw)
    res = orc.solve(d)
    full_nnz = _full_kkt_nnz(workload)
    scale = full_nnz / configs.kkt_nnz(d)
    text = (f"{key} {sample_kw}: KKT nnz {configs.kkt_nnz(d)} of {full_nnz} (1/{scale:.0f}), full solve, "
            f"{res.iterations} iterations, status {res.status}; seconds scaled linearly in KKT nnz to the full "
            f"workload (the CPU factorisation grows at least linearly, so this under-states the CPU time)")
    return res.setup_seconds, res.solve_seconds, res.iterations, scale, text


_NNZ_CACHE = {}


def _full_kkt_nnz(workload):
    if workload not in _NNZ_CACHE:
        key, full_kw, _ = WORKLOADS[workload]
        if key == "C4_group_lasso":  # closed form, avoids generating the full problem in the CPU arm
            rng = np.random.default_rng(0)
            q = rng.integers(full_kw["qlo"], full_kw["qhi"] + 1, full_kw["groups"])
            nf = int((q - 1).sum())
            ns = full_kw["samples"]
            n = nf + ns + full_kw["groups"]
            _NNZ_CACHE[workload] = int(n + nf * full_kw["nnz_per_col"] + ns + ns + (nf + full_kw["groups"])
                                       + (q * (q + 1) // 2).sum())
        else:
            from paper_2603_29197_b200 import configs

            _NNZ_CACHE[workload] = configs.kkt_nnz(configs.make(key, **full_kw))
    return _NNZ_CACHE[workload]


def run_reference(args):
    """--impl reference: the reference's CPU path (the pinned C/NumPy port of it --
    the numba reference itself does not exist on the GPU box) on the host cores."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    from oracle import qsocp_oracle as orc

    orc.build()
    times, e2e = [], []
    text = ""
    for k in range(args.warmup + args.steps):
        st, so, iters, scale, text = cpu_solve_sample(args.workload)
        if k >= args.warmup:
            times.append(so * scale)
            e2e.append((st + so) * scale)
    val = float(np.mean(times))
    key, full_kw, _ = WORKLOADS[args.workload]
    line = {
        "impl": "reference", "metric": "ipm_solve_seconds", "value": val, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": val * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, **full_kw},
        "cpu_baseline": {"value": val, "unit": "s", "cores": 1, "kind": "port", "sample": text},
        "e2e": {"value": float(np.mean(e2e)), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


# ------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch

    rank, local_rank, world = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_2603_29197_b200 as qs
    from paper_2603_29197_b200 import configs
    from paper_2603_29197_b200.ipm import DeviceSolver
    from paper_2603_29197_b200.problem import Settings, SolveStatus

    key, full_kw, _ = WORKLOADS[args.workload]
    data = configs.make(key, seed=rank, **full_kw)
    settings = Settings(device=local_rank)
    hbm_peak, peak_src = peaks()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    # ---- resident arm: setup once, time K solves with CUDA events on the device
    t0 = time.perf_counter()
    dev = DeviceSolver(data, settings)
    dev.set_stream(torch.cuda.current_stream().cuda_stream)  # so torch.cuda.Event brackets the library's launches
    setup_seconds = time.perf_counter() - t0
    for _ in range(args.warmup):
        status, iters, _ = dev.run()
        assert status is SolveStatus.SOLVED, status
    f0, s0, l0 = dev.counters()
    tm0 = dev.timers()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    # the handle launches on its own stream; bracket with full-device synchronisation
    t_start = time.perf_counter()
    ev[0].record()
    iters_total = 0
    for _ in range(args.steps):
        status, iters, it = dev.run()
        iters_total += iters
    ev[1].record()
    barrier()
    wall = time.perf_counter() - t_start
    dev_seconds = ev[0].elapsed_time(ev[1]) * 1e-3
    f1, s1, l1 = dev.counters()
    tm1 = dev.timers()
    clocks = sampler.stop() if sampler else None
    per_solve = dev_seconds / args.steps
    phase = {k: (tm1[k] - tm0[k]) / args.steps for k in tm1 if k in tm0}

    # ---- roofline of the dominant hot-path kernel + the other hot-path kernels (CUDA events in the library)
    cone = data.cone
    m, l, nsoc = cone.total_dim, cone.orthant_dim, cone.soc_count
    S = l + sum(q * (q + 1) // 2 for q in cone.soc_dims)
    n, p = data.n, data.p
    nnz_pag = 2 * data.P.nnz + 2 * data.A.nnz + 2 * data.G.nnz
    # fused kernels are scored against the un-fused algorithmic bytes of the logical ops they cover
    kernels = [(1, "neg_wtw_scatter", 8 * S + 8 * (m + nsoc)),
               (0, "nt_scaling+lam_sq+pred_rhs_cone", 40 * m + 8 * (l + nsoc) + 64 * m),
               (4, "post_solve(pred)+mu_aff", 80 * m + 32 * m), (6, "dcomp+corr_rhs_cone", 80 * m + 64 * m),
               (5, "post_solve(corr)", 80 * m), (15, "update_iterate", 24 * (n + p) + 48 * m),
               (7, "residuals", 12 * nnz_pag + 8 * (3 * n + 2 * p + 4 * m))]
    kt = {}
    for kid, name, nbytes in kernels:
        ms = dev.time_kernel(kid, 20)
        msc = dev.time_kernel(kid, 10, cold=True)  # L2 flushed before every launch
        kt[name] = {"us": ms * 1e3, "alg_bytes": nbytes, "gbs": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / hbm_peak,
                    "cold_us": msc * 1e3, "cold_frac": nbytes / msc / 1e6 / hbm_peak}
    dom = kt["neg_wtw_scatter"]
    iters_per = iters_total / args.steps
    # the dominant kernel inside the timed region: the kkt_update phase (CUDA events in the library around the
    # prepass + scatter launches) runs once per factorisation = iterations + 1 times per solve
    dom_launches = iters_per + 1
    dom_us_region = phase.get("kkt_update", 0.0) / max(dom_launches, 1) * 1e6
    if dom_us_region > 0:
        dom = dict(dom, us_isolated=dom["us"], us=dom_us_region, gbs=dom["alg_bytes"] / dom_us_region / 1e3,
                   frac=dom["alg_bytes"] / dom_us_region / 1e3 / hbm_peak)
    cone_kkt_us = (phase.get("cone", 0.0) + phase.get("kkt_update", 0.0)) / max(iters_per, 1) * 1e6
    alg_iter = 8 * S + 576 * m + 32 * (n + p + m) + 24 * (n + p)  # un-fused algorithmic bytes per iteration
    fstats = dev.factor_stats()
    dev.close()

    # ---- end-to-end arm: the public API on host buffers (setup + solve + result read-back), every step
    def e2e_once():
        res = qs.Solver("cuda").setup(data.n, data.m, data.p, data.P, data.c, data.A, data.b, data.G, data.h,
                                      cone.orthant_dim, cone.soc_count, cone.soc_dims, device=local_rank).solve()
        assert res.status is SolveStatus.SOLVED
        return res

    e2e_s = float("nan")
    if args.e2e_steps > 0:  # 0 = skip (profiling runs only; a bench line without e2e is not a result)
        e2e_once()  # warm-up
        barrier()
        te = time.perf_counter()
        for _ in range(args.e2e_steps):
            res = e2e_once()
        barrier()
        e2e_s = (time.perf_counter() - te) / args.e2e_steps
    # bytes per e2e step, counted by the library from the buffers it copies: host -> device = row views of P/A/G
    # (int32 index + fp64 value), c/b/h, the KKT column pointers and the analysis structures (the KKT entries are
    # written by the device); device -> host = the scalar block of every phase and x, y, z, s at the end
    if args.e2e_steps > 0:
        h2d, d2h = res.timers["h2d_bytes"], res.timers["d2h_bytes"]
    else:
        h2d = d2h = 0
    knnz = configs.kkt_nnz(data)

    if world > 1:
        t = torch.tensor([per_solve, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per_solve, e2e_s = t.tolist()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        from oracle import qsocp_oracle as orc

        orc.build()
        st, so, ci, scale, text = cpu_solve_sample(args.workload)
        cpu = {"value": so * scale, "unit": "s", "cores": 1, "kind": "port", "sample": text,
               "sample_seconds": so, "sample_setup_seconds": st, "scale": scale,
               "e2e_value": (st + so) * scale}
    line = {
        "metric": "ipm_solve_seconds", "value": per_solve, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_solve * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, **full_kw, "n": n, "p": p, "m": m, "kkt_nnz": configs.kkt_nnz(data),
                   "l2": "inputs larger than L2 (KKT values 0.97 GB, factor 5.7 GB are rewritten every iteration)"},
        "iterations_per_solve": iters_per, "host_wall_seconds_per_solve": wall / args.steps,
        "e2e": {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "setup_seconds_resident_arm": setup_seconds},
        "gpu_launches": int(l1 - l0),
        "roofline": {"bound": "hbm", "kernel": "k_neg_wtw<DIRECT> (-W'W generate + scatter into K.values)",
                     "achieved": dom["gbs"], "peak": hbm_peak, "unit": "GB/s", "frac": dom["frac"],
                     "peak_source": peak_src, "traffic": args.traffic, "alg_bytes_per_launch": dom["alg_bytes"],
                     "us_per_launch": dom["us"], "us_per_launch_isolated": dom.get("us_isolated", dom["us"]),
                     "timing": "CUDA events around the KKT-update phase of every factorisation inside the timed solves "
                               "(prepass + scatter); 'isolated' = 20 back-to-back launches after the timed region"},
        "hot_path": {"cone_plus_kkt_update_us_per_iter": cone_kkt_us, "alg_bytes_per_iter": alg_iter,
                     "frac_of_hbm_peak_unfused_alg": alg_iter / max(cone_kkt_us, 1e-9) / 1e3 / hbm_peak,
                     "kernels": kt},
        "phase_seconds_per_solve": phase,
        "factor": {k: fstats[k] for k in ("supernodes", "levels", "L_nnz", "factor_flops", "max_front_rows")},
        "clocks": clocks,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C4_group_lasso", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the dominant kernel from the committed ncu capture")
    args = ap.parse_args()
    if args.traffic is None:
        tr = os.path.join(ROOT, "profiles", "dominant_kernel_traffic.json")
        if os.path.exists(tr):
            args.traffic = json.load(open(tr)).get(args.workload)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
