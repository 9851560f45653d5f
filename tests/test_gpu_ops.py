"""GPU parity of the operator surface (kernels.py mirror) against the
reference's golden outputs and the oracle.  Bitwise wherever the reference
is bitwise (kernels.py:1-7); tolerance only for tree-order dots."""

from __future__ import annotations

import types

import numpy as np
import pytest

import oracle
from conftest import golden_matrix, load_golden, python_dot

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_2105_06176_b200")
torch = pytest.importorskip("torch")
from paper_2105_06176_b200 import _lib  # noqa: E402

NAMES = ("z", "q", "s", "p", "x", "r", "u", "w", "m", "n")


@pytest.fixture(scope="module")
def K(cuda):
    return load_golden("kernels.npz")


def test_fused_update_bitwise_golden(K):
    st = types.SimpleNamespace(**{nm: K["in_" + nm].copy() for nm in NAMES})
    pb.fused_pipecg_update(st, float(K["alpha"]), float(K["beta"]))
    for nm in NAMES:
        np.testing.assert_array_equal(getattr(st, nm), K["out_" + nm], err_msg=nm)


def test_fused_update_bitwise_device_tensors(K):
    st = types.SimpleNamespace(**{nm: torch.from_numpy(K["in_" + nm].copy()).cuda() for nm in NAMES})
    pb.fused_pipecg_update(st, float(K["alpha"]), float(K["beta"]))
    for nm in NAMES:
        np.testing.assert_array_equal(getattr(st, nm).cpu().numpy(), K["out_" + nm], err_msg=nm)


@pytest.mark.parametrize("n", [1, 2, 31, 257, 100003])
def test_fused_update_bitwise_random_sizes(cuda, n):
    rng = np.random.default_rng(n)
    v = {nm: rng.standard_normal(n) * 10.0 ** rng.integers(-4, 5, n) for nm in NAMES}
    alpha, beta = rng.uniform(-8, 8), rng.uniform(-8, 8)
    exp = oracle.fused_update(v, alpha, beta)
    st = types.SimpleNamespace(**{k: a.copy() for k, a in v.items()})
    pb.fused_pipecg_update(st, alpha, beta)
    for nm in NAMES:
        np.testing.assert_array_equal(getattr(st, nm), exp[nm], err_msg=nm)


def test_dot_seq_bitwise(K):
    a, b = K["dot_a"], K["dot_b"]
    assert pb.dot(a, b) == float(K["dot_ab"]) == python_dot(a, b)
    assert pb.norm2(a) == np.sqrt(pb.dot(a, a))


def test_dot_tree_close_and_deterministic(K):
    rng = np.random.default_rng(3)
    a = rng.standard_normal(1_000_003)
    b = rng.standard_normal(1_000_003)
    ref = oracle.dot(a, b)
    t1 = pb.dot(a, b, mode="tree")
    t2 = pb.dot(a, b, mode="tree")
    assert t1 == t2
    assert abs(t1 - ref) <= 1e-12 * np.sum(np.abs(a * b))


def test_dot_length_mismatch(cuda):
    with pytest.raises(ValueError):
        pb.dot(np.ones(3), np.ones(4))


def test_spmv_bitwise_p125_golden(K):
    A = golden_matrix(K, "p125n6")
    np.testing.assert_array_equal(pb.spmv(A, K["p125n6_x"]), K["p125n6_y"])


def test_spmv_bitwise_rectangular_golden(K):
    A = golden_matrix(K, "rand")
    Am = pb.CsrMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, A.values)
    np.testing.assert_array_equal(pb.spmv(Am, K["rand_x"]), K["rand_y"])


def test_spmv_out_and_validation(cuda):
    I4 = pb.csr_from_dense(np.eye(4))
    x = np.arange(4.0)
    out = np.empty(4)
    got = pb.spmv(I4, x, out=out)
    assert got is out
    np.testing.assert_array_equal(out, x)
    with pytest.raises(ValueError):
        pb.spmv(I4, np.ones(5))
    with pytest.raises(ValueError):
        pb.spmv(I4, np.ones(4), out=np.empty(3))


@pytest.mark.parametrize("kind,n", [("2d5", 64), ("3d7", 20), ("3d27", 12), ("p125", 7)])
def test_spmv_stencils_bitwise_vs_oracle(cuda, kind, n):
    A = oracle.stencil(kind, n)
    x = np.random.default_rng(5).standard_normal(A.n_rows)
    np.testing.assert_array_equal(pb.spmv(A, x), oracle.spmv(A, x))


def test_spmv_long_rows_close(cuda):
    # an arrow matrix: row 0 and column 0 dense -> row 0 takes the block path
    n = 5000
    rows = [0] * n + list(range(1, n)) + list(range(1, n))
    cols = list(range(n)) + [0] * (n - 1) + list(range(1, n))
    vals = np.concatenate([np.full(n, -1.0), np.full(n - 1, -1.0), np.full(n - 1, 4.0)])
    vals[0] = float(n)
    import scipy.sparse as sp

    S = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    S.sort_indices()
    A = pb.CsrMatrix(n, n, S.indptr, S.indices, S.data)
    x = np.random.default_rng(9).standard_normal(n)
    y = pb.spmv(A, x)
    ref = oracle.spmv(A, x)
    np.testing.assert_array_equal(y[1:], ref[1:])
    assert abs(y[0] - ref[0]) <= 1e-12 * np.sum(np.abs(S.data[:n] * x))


def test_stencil_device_matches_oracle(cuda):
    for kind, n in (("2d5", 33), ("3d7", 11), ("3d27", 9), ("p125", 7)):
        d = pb.stencil_device(kind, n).to_host()
        o = oracle.stencil(kind, n)
        np.testing.assert_array_equal(d.row_offsets, o.row_offsets)
        np.testing.assert_array_equal(d.col_indices, o.col_indices)
        np.testing.assert_array_equal(d.values, o.values)


def test_stencil_device_row_block(cuda):
    full = pb.stencil_device("3d7", 10).to_host()
    blk = pb.stencil_device("3d7", 10, 230, 611)
    h = blk.to_host() if False else None
    ro = blk.rowptr[: blk.n_rows + 1].cpu().numpy().astype(np.int64)
    base = full.row_offsets[230]
    np.testing.assert_array_equal(ro + base, full.row_offsets[230:612])
    np.testing.assert_array_equal(blk.col[: blk.nnz].cpu().numpy(),
                                  full.col_indices[base: full.row_offsets[611]])
    del h


def test_jacobi_setup_and_apply(K):
    A = golden_matrix(K, "p125n6")
    pc = pb.jacobi_setup(A)
    np.testing.assert_array_equal(pc.inv_diag, K["p125n6_inv_diag"])
    np.testing.assert_array_equal(pb.jacobi_apply(pc, K["p125n6_x"]), K["p125n6_jacobi"])
    out = np.empty(A.n_rows)
    assert pb.jacobi_apply(pc, K["p125n6_x"], out=out) is out


def test_jacobi_errors(cuda):
    with pytest.raises(ValueError, match="row 1: missing diagonal"):
        pb.jacobi_setup(pb.csr_from_dense(np.array([[1.0, 1.0], [1.0, 0.0]])))
    with pytest.raises(ValueError, match="zero diagonal"):
        pb.jacobi_setup(pb.CsrMatrix(2, 2, [0, 1, 2], [0, 1], [1.0, 0.0]))
    with pytest.raises(ValueError):
        pb.jacobi_setup(pb.csr_from_dense(np.ones((2, 3))))


def test_fused_update_pc_dots(cuda):
    rng = np.random.default_rng(77)
    n = 300001
    v = {nm: rng.standard_normal(n) for nm in NAMES}
    d = rng.uniform(0.1, 1.0, n)
    alpha, beta = 0.37, 0.81
    exp = oracle.fused_update(v, alpha, beta)
    st = types.SimpleNamespace(**{k: torch.from_numpy(a.copy()).cuda() for k, a in v.items()})
    g, dl, uu = pb.fused_pipecg_update_pc_dots(st, torch.from_numpy(d).cuda(), alpha, beta)
    for nm in ("z", "q", "s", "p", "x", "r", "u", "w"):
        np.testing.assert_array_equal(getattr(st, nm).cpu().numpy(), exp[nm], err_msg=nm)
    np.testing.assert_array_equal(st.m.cpu().numpy(), d * exp["w"])
    for got, (a, b) in zip((g, dl, uu), ((exp["r"], exp["u"]), (exp["w"], exp["u"]),
                                          (exp["u"], exp["u"]))):
        assert abs(got - oracle.dot(a, b)) <= 1e-12 * np.sum(np.abs(a * b))


def test_host_transfer_pipeline(cuda):
    """csrc/hostio.cu: chunked pinned-ring uploads (with int64 -> int32
    narrowing) and downloads, across several 8 MB ring slots."""
    from paper_2105_06176_b200._device import d2h, h2d

    n = (32 << 20) // 4 * 3 + 12345  # > 2 ring slots of narrowed data
    rng = np.random.default_rng(5)
    idx = rng.integers(-2**31, 2**31, size=n, dtype=np.int64)
    dst = torch.empty(n, dtype=torch.int32, device="cuda")
    h2d(dst, idx, narrow=True)
    np.testing.assert_array_equal(dst.cpu().numpy(), idx.astype(np.int32))
    vals = rng.standard_normal(n // 2 + 7)
    dv = torch.empty(vals.size, dtype=torch.float64, device="cuda")
    h2d(dv, vals)
    np.testing.assert_array_equal(d2h(dv), vals)
    bad = idx.copy()
    bad[n - 3] = 2**31  # outside int32
    with pytest.raises(_lib.NativeError) as e:
        h2d(dst, bad, narrow=True)
    assert e.value.code == _lib.PCG_ERANGE


def test_host_transfer_pipeline_interleaved(cuda):
    """pipecg_b200_h2d_multi: several arrays of mixed kinds (narrowed
    indices, copied values, an empty one) interleaved chunk by chunk land
    exactly where single transfers would; an out-of-range index anywhere
    still raises PCG_ERANGE."""
    from paper_2105_06176_b200._device import h2d_multi

    rng = np.random.default_rng(9)
    n1, n2, n3 = (8 << 20) // 4 * 5 + 321, (8 << 20) // 8 * 3 + 17, 1000
    a1 = rng.integers(-2**31, 2**31, size=n1, dtype=np.int64)
    a2 = rng.standard_normal(n2)
    a3 = rng.integers(0, 100, size=n3, dtype=np.int64)
    d1 = torch.empty(n1, dtype=torch.int32, device="cuda")
    d2 = torch.empty(n2, dtype=torch.float64, device="cuda")
    d3 = torch.empty(n3, dtype=torch.int32, device="cuda")
    d0 = torch.empty(0, dtype=torch.float64, device="cuda")
    h2d_multi([(d1, a1, True), (d0, np.zeros(0), False), (d2, a2, False), (d3, a3, True)])
    torch.cuda.synchronize()
    np.testing.assert_array_equal(d1.cpu().numpy(), a1.astype(np.int32))
    np.testing.assert_array_equal(d2.cpu().numpy(), a2)
    np.testing.assert_array_equal(d3.cpu().numpy(), a3.astype(np.int32))
    bad = a3.copy()
    bad[-1] = -2**31 - 1
    with pytest.raises(_lib.NativeError) as e:
        h2d_multi([(d2, a2, False), (d3, bad, True)])
    assert e.value.code == _lib.PCG_ERANGE
