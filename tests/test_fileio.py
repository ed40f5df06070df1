"""Problem files: the reference's QOCOPROB 1 text form and the binary, mappable QOCOPROB 2 form."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from util import GOLDEN, load_golden, problem_from_golden
from paper_2603_29197_b200 import configs, fileio
from paper_2603_29197_b200.errors import BadSparseStructure

REF_FILE = os.path.join(GOLDEN, "portfolio_4.qocoprob")  # written by the reference's save_problem (oracle/gen_golden.py)


def same_problem(a, b):
    assert (a.n, a.m, a.p) == (b.n, b.m, b.p)
    assert a.cone.orthant_dim == b.cone.orthant_dim and tuple(a.cone.soc_dims) == tuple(b.cone.soc_dims)
    for k in "PAG":
        A, B = getattr(a, k), getattr(b, k)
        assert (A.rows, A.cols) == (B.rows, B.cols)
        assert np.array_equal(A.col_pointers, B.col_pointers) and np.array_equal(A.row_indices, B.row_indices)
        assert np.array_equal(A.values, B.values)
    for k in "cbh":
        assert np.array_equal(getattr(a, k), getattr(b, k))


def test_text_file_written_by_the_reference_loads_bit_exact():
    d = problem_from_golden(load_golden("portfolio_4"))
    same_problem(fileio.load_problem(REF_FILE), d)
    # and the writer reproduces the reference's text byte for byte
    assert fileio.problem_to_text(d) == open(REF_FILE).read()


def test_text_errors_match_reference_types(tmp_path):
    text = open(REF_FILE).read()
    with pytest.raises(BadSparseStructure):
        fileio.problem_from_text(text.replace("QOCOPROB 1", "QOCOPROB 9", 1))
    with pytest.raises(BadSparseStructure):
        fileio.problem_from_text(text[: len(text) // 2])
    with pytest.raises(BadSparseStructure):
        fileio.problem_from_text(text.replace("MAT A", "MAT Q", 1))


@pytest.mark.parametrize("make", [lambda: configs.make("C1_random_qp", small=True), lambda: configs.make("C4_group_lasso", small=True),
                                  lambda: configs.make("C5_mpc", small=True), lambda: problem_from_golden(load_golden("tiny_qp")),
                                  lambda: problem_from_golden(load_golden("soc_slice"))])
def test_binary_round_trip_and_mapping(tmp_path, make):
    d = make()
    path = tmp_path / "p.qp2"
    perm = np.random.default_rng(0).permutation(d.n + d.p + d.m)
    fileio.save_problem(d, path, perm=perm, meta={"generator": "test", "seed": 0})
    pf = fileio.ProblemFile(path)
    same_problem(pf.data, d)
    assert np.array_equal(pf.perm, perm) and pf.meta == {"generator": "test", "seed": 0}
    # arrays are views of the mapping (no parse, no copy), aligned for 128-bit loads / pinned DMA
    for a in (pf.data.G.values, pf.data.G.row_indices, pf.data.c, pf.data.h):
        if a.size:
            assert not a.flags.owndata and a.ctypes.data % 64 == 0 and not a.flags.writeable
    same_problem(fileio.load_problem(path), d)  # front end detects the form
    # text -> binary -> text
    t = tmp_path / "p.qocoprob"
    fileio.save_problem(d, t)
    same_problem(fileio.load_problem(t), d)


def test_binary_rejects_damaged_files(tmp_path):
    d = configs.make("C5_mpc", small=True)
    path = tmp_path / "p.qp2"
    fileio.save_problem(d, path)
    blob = open(path, "rb").read()
    (tmp_path / "cut.qp2").write_bytes(blob[: len(blob) - 4096])
    with pytest.raises(BadSparseStructure):
        fileio.ProblemFile(tmp_path / "cut.qp2")
    (tmp_path / "magic.qp2").write_bytes(b"QOCOPROB 3\n" + blob[11:])
    with pytest.raises(BadSparseStructure):
        fileio.ProblemFile(tmp_path / "magic.qp2")


def test_cli_info_and_convert(tmp_path):
    env = dict(os.environ, PYTHONPATH=os.path.dirname(os.path.dirname(GOLDEN)))
    out = subprocess.run([sys.executable, "-m", "paper_2603_29197_b200", "info", "--in", REF_FILE], env=env,
                         check=True, capture_output=True, text=True).stdout
    info = json.loads(out)
    d = problem_from_golden(load_golden("portfolio_4"))
    assert info["n"] == d.n and info["m"] == d.m and info["soc_dims"] == list(d.cone.soc_dims)
    q = tmp_path / "x.qp2"
    subprocess.run([sys.executable, "-m", "paper_2603_29197_b200", "convert", "--in", REF_FILE, "--out", str(q)],
                   env=env, check=True)
    same_problem(fileio.load_problem(q), d)


@pytest.mark.gpu
def test_cli_solve_from_binary_file_matches_reference_golden(tmp_path):
    """cli.py:35-52 with --backend cuda: the JSON payload of the reference's CLI, values within the parity bar."""
    g = load_golden("portfolio_4")
    d = problem_from_golden(g)
    q = tmp_path / "x.qp2"
    fileio.save_problem(d, q)
    env = dict(os.environ, PYTHONPATH=os.path.dirname(os.path.dirname(GOLDEN)))
    r = subprocess.run([sys.executable, "-m", "paper_2603_29197_b200", "solve", "--in", str(q), "--backend", "cuda",
                        "--pin"], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    res = json.loads(r.stdout)
    assert res["status"] == "Solved" and abs(res["iterations"] - int(g["iterations"])) <= 1
    assert abs(res["objective"] - float(g["objective"])) <= 1e-6 * max(1.0, abs(float(g["objective"])))
    assert np.max(np.abs(np.array(res["x"]) - g["x"])) <= 1e-5 * max(1.0, np.max(np.abs(g["x"])))
