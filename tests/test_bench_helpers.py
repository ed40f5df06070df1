"""Host-side pieces of bench.py (no GPU): workload / ladder tables, the offline CPU records the ladder cites, and the
reference arm's contract (complete solves of a ladder rung, oracle library only)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_workload_has_a_ladder_of_smaller_instances_of_the_same_generator():
    import bench
    from paper_2603_29197_b200 import configs

    assert set(bench.LADDERS) == set(bench.WORKLOADS)
    key, full = bench.WORKLOADS["C4_group_lasso"]
    rungs = bench.LADDERS["C4_group_lasso"]
    assert [r[0] for r in rungs] == ["1/100", "1/32", "1/10"]
    sizes = [configs.kkt_nnz(configs.make(key, **kw)) for _, kw in rungs[:2]]
    assert sizes[0] < sizes[1] < 1.3e8 and all(kw["qlo"] == full["qlo"] and kw["qhi"] == full["qhi"] for _, kw in rungs)


def test_offline_cpu_records_are_the_committed_oracle_runs():
    import bench

    full = bench.offline_record("C4_group_lasso", "full")
    assert full["status"] == "Solved" and full["iterations"] == 14 and full["solve_seconds"] > 1000
    assert "offline" in full["source"] and full["host"]["threads_used"] == 1
    tenth = bench.offline_record("C4_group_lasso", "1/10")
    assert tenth["iterations"] == 11 and "reference AMD" in tenth["ordering"]
    assert bench.offline_record("C5_mpc", "full") is None  # no committed run: the ladder says so instead of guessing


def test_reference_arm_prints_a_measured_lower_bound_and_maps_only_the_oracle(oracle):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          "C5_mpc", "--steps", "1", "--warmup", "0", "--ref-budget", "30"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["lower_bound"] is True and line["higher_is_better"] is False
    assert line["native_libraries_mapped"] == ["oracle/liboracle.so"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] == 1
    assert line["value"] == line["cpu_baseline"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["ladder"][0]["status"] == "Solved" and line["ladder"][0]["cpu_source"] == "measured in this run"
    assert line["config"]["workload"] == "C5_mpc"
