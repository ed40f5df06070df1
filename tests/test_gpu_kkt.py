"""GPU parity of the KKT scaling-block update and the sparse products."""

import ctypes as C

import numpy as np
import pytest

from paper_2603_29197_b200 import _lib
from paper_2603_29197_b200.cones import DeviceCones, identity_scaling
from paper_2603_29197_b200.kkt import assemble_kkt
from util import golden_problem_names, load_golden, problem_from_golden, random_interior_point

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", golden_problem_names())
def test_write_scaling_vs_oracle(oracle, name):
    g = load_golden(name)
    d = problem_from_golden(g)
    rng = np.random.default_rng(1)
    s, z = random_interior_point(d.cone, rng), random_interior_point(d.cone, rng)
    ref_kkt = oracle.assemble_kkt(d)
    sc = oracle.compute_nt_scaling(s, z, d.cone)
    oracle.write_scaling(ref_kkt, sc)
    dc = DeviceCones(d.cone)
    for direct in (False, True):
        kkt = assemble_kkt(d)
        before = kkt.matrix.values.copy()
        dc.write_scaling(kkt, sc, direct=direct)
        assert np.allclose(kkt.matrix.values, ref_kkt.matrix.values, rtol=1e-12, atol=0)
        # only mapped entries change (test_kkt.py:94-104)
        mask = np.ones(before.size, bool)
        mask[kkt.nt_entry_positions] = False
        assert np.array_equal(kkt.matrix.values[mask], before[mask])
    # identity update is a no-op on the assembled values (test_kkt.py:79-84)
    kkt = assemble_kkt(d)
    before = kkt.matrix.values.copy()
    dc.write_scaling(kkt, identity_scaling(d.cone))
    assert np.array_equal(kkt.matrix.values, before)
    dc.close()


@pytest.mark.parametrize("name", ["huber_20", "portfolio_4", "random_1", "tv_denoising_8"])
def test_spmv_vs_reference_golden(name):
    import torch

    g = load_golden(name)
    d = problem_from_golden(g)
    lib = _lib.require_device(0)
    h = lib.qs_create(0)
    dev = torch.device("cuda", 0)

    def csr_of(M, transpose):
        import scipy.sparse as sp

        S = sp.csc_matrix((M.values, M.row_indices, M.col_pointers), shape=(M.rows, M.cols))
        S = (S.T if transpose else S).tocsr()
        S.sort_indices()
        return S

    def gpu_spmv(S, x):
        ptr = torch.as_tensor(S.indptr.astype(np.int32)).to(dev)
        idx = torch.as_tensor(S.indices.astype(np.int32)).to(dev)
        val = torch.as_tensor(S.data.astype(np.float64)).to(dev)
        xd = torch.as_tensor(x).to(dev)
        y = torch.zeros(max(S.shape[0], 1), dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        rc = lib.qs_spmv_csr(h, S.shape[0], S.shape[1], C.c_void_p(ptr.data_ptr()), C.c_void_p(idx.data_ptr()),
                             C.c_void_p(val.data_ptr()), C.c_void_p(xd.data_ptr()), C.c_void_p(y.data_ptr()), 0)
        _lib.check(lib, h, rc)
        lib.qs_sync(h)
        return y[: S.shape[0]].cpu().numpy()

    x, y, z = g["spmv_x"], g["spmv_y"], g["spmv_z"]
    for M, tr, vec, key in ((d.A, False, x, "Ax"), (d.G, False, x, "Gx"), (d.A, True, y, "Aty"), (d.G, True, z, "Gtz")):
        if M.rows == 0:
            continue
        got = gpu_spmv(csr_of(M, tr), vec)
        assert np.allclose(got, g[key], rtol=1e-13, atol=1e-13 * np.max(np.abs(g[key]), initial=1.0)), key
    # literal symmetric product over the stored upper triangle of K (sparse.py:143-150)
    K_p = torch.as_tensor(g["K_p"]).to(dev)
    K_i = torch.as_tensor(g["K_i"].astype(np.int32)).to(dev)
    K_x = torch.as_tensor(g["K_x"]).to(dev)
    v = torch.as_tensor(g["kkt_vec"]).to(dev)
    out = torch.zeros(v.numel(), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    rc = lib.qs_spmv_sym_upper(h, v.numel(), C.c_void_p(K_p.data_ptr()), C.c_void_p(K_i.data_ptr()),
                               C.c_void_p(K_x.data_ptr()), C.c_void_p(v.data_ptr()), C.c_void_p(out.data_ptr()))
    _lib.check(lib, h, rc)
    lib.qs_sync(h)
    ref = g["K_times_vec"]
    assert np.allclose(out.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.max(np.abs(ref)))
    lib.qs_destroy(h)


def test_spmv_long_rows_cta_per_row():
    """Rows of >= 512 entries on average take the CTA-per-row path of the gather products (spmv_kernels.cu)."""
    import scipy.sparse as sp
    import torch

    rng = np.random.default_rng(5)
    rows, cols = 37, 6000
    S = sp.random(rows, cols, density=0.15, random_state=7, format="csr", dtype=np.float64)  # ~900 per row
    S.sort_indices()
    x = rng.standard_normal(cols)
    lib = _lib.require_device(0)
    h = lib.qs_create(0)
    dev = torch.device("cuda", 0)
    ptr = torch.as_tensor(S.indptr.astype(np.int32)).to(dev)
    idx = torch.as_tensor(S.indices.astype(np.int32)).to(dev)
    val = torch.as_tensor(S.data).to(dev)
    xd = torch.as_tensor(x).to(dev)
    y = torch.ones(rows, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    for accumulate, base in ((0, 0.0), (1, 1.0)):
        y.fill_(1.0)
        torch.cuda.synchronize()
        rc = lib.qs_spmv_csr(h, rows, cols, C.c_void_p(ptr.data_ptr()), C.c_void_p(idx.data_ptr()),
                             C.c_void_p(val.data_ptr()), C.c_void_p(xd.data_ptr()), C.c_void_p(y.data_ptr()), accumulate)
        _lib.check(lib, h, rc)
        lib.qs_sync(h)
        ref = S @ x + base
        assert np.allclose(y.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.max(np.abs(ref)))
    lib.qs_destroy(h)
