"""Irregular matrices (BASELINE.json configs[3]: power-law row lengths) on
the nnz-balanced fused variant D, checked against the oracle.

* Rows staged in shared memory are summed in CSR order from the products
  a_k * m[c_k], so with dot_mode="seq" a solve without hub rows is bitwise
  the reference's (kernels.py:64-70, solvers.py:324-387), whatever the tile
  boundaries are.
* Hub rows (longer than the tile's hub threshold) are combined with a
  fixed tree: graded against the oracle's own reorder envelope.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_2105_06176_b200")
from test_gpu_solver import assert_within_envelope, envelope  # noqa: E402

VARIANTS = ["fused-d", "two", "fused-g"]


def _problem(A):
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    return b, x0, d, tol


def _random_spd(n, max_len, seed):
    """Symmetric, strictly diagonally dominant, row lengths 1..max_len."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len // 2, size=n)
    r = np.repeat(np.arange(n), lens)
    c = rng.integers(0, n, size=r.size)
    keep = r != c
    r, c = r[keep], c[keep]
    dense_key = np.unique(np.minimum(r, c) * n + np.maximum(r, c))
    a, b = dense_key // n, dense_key % n
    v = -rng.uniform(0.1, 1.0, size=a.size)
    rows = np.concatenate([a, b, np.arange(n)])
    cols = np.concatenate([b, a, np.arange(n)])
    vals = np.concatenate([v, v, np.zeros(n)])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    diag = np.bincount(rows, weights=np.abs(vals), minlength=n) + 1.0
    vals[rows == cols] = diag
    ro = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ro[1:])
    return pb.CsrMatrix(n, n, ro, cols, vals)


@pytest.mark.parametrize("engine", VARIANTS)
@pytest.mark.parametrize("dcap", [None, 512, 2048])
def test_powerlaw_seq_bitwise_balanced_tiles(cuda, monkeypatch, dcap, engine):
    """nnz-capped tiles, every row <= 256 nonzeros (so the init SpMVs take
    the in-order row path too) and no hub tiles: bitwise in seq-dot mode."""
    if dcap:
        monkeypatch.setenv("PIPECG_B200_DCAP", str(dcap))
    A = pb.generate_powerlaw(2**12)
    assert A.row_nnz().max() <= min(256, (dcap or 10**9) // 2)
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=2000)
    pc = pb.jacobi_setup(A)
    np.testing.assert_array_equal(pc.inv_diag, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=2000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pc, cfg,
                             options=pb.DeviceOptions(dot_mode="seq", engine=engine))
    assert rep.iterations == ref.iterations
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)


@pytest.mark.parametrize("engine", ["auto", "fused-d", "two", "fused-g"])
def test_powerlaw_tree_within_envelope(cuda, engine):
    A = pb.generate_powerlaw(2**16)
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=2000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=2000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                             options=pb.DeviceOptions(engine=engine))
    assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x,
                           envelope(A, b, x0, d, tol, 2000))


@pytest.mark.parametrize("engine", VARIANTS)
@pytest.mark.parametrize("dcap", [64, 256])
def test_powerlaw_hub_rows(cuda, monkeypatch, dcap, engine):
    """A small tile cap turns the long rows into hub tiles (tree-combined)."""
    monkeypatch.setenv("PIPECG_B200_DCAP", str(dcap))
    A = pb.generate_powerlaw(2**15)
    assert A.row_nnz().max() > dcap // 2  # hubs exist
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=2000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=2000, record_history=True)
    env = envelope(A, b, x0, d, tol, 2000)
    for mode in ("tree", "seq"):
        x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                                 options=pb.DeviceOptions(engine=engine, dot_mode=mode))
        assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x, env)


@pytest.mark.parametrize("engine", VARIANTS)
@pytest.mark.parametrize("dcap,max_len", [(16, 12), (64, 40), (1000, 200)])
def test_random_spd_tiles_bitwise(cuda, monkeypatch, dcap, max_len, engine):
    """Ragged rows and many tile splits: bitwise when no row is a hub
    (every row <= dcap/2 nonzeros), else within the reorder envelope."""
    monkeypatch.setenv("PIPECG_B200_DCAP", str(dcap))
    A = _random_spd(5000, max_len, seed=dcap)
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                             options=pb.DeviceOptions(dot_mode="seq", engine=engine))
    if A.row_nnz().max() <= dcap // 2:
        assert rep.history == ref.history
        np.testing.assert_array_equal(x, ref.x)
    else:
        assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x,
                               envelope(A, b, x0, d, tol, 3000))


@pytest.mark.parametrize("engine", ["two", "fused-g"])
@pytest.mark.parametrize("n", [2**12, 3000])
def test_sell_layout_bitwise(cuda, monkeypatch, n, engine):
    """Engine 2's SELL-C-sigma SpMV (rows length-sorted inside 1024-row
    windows, 32-row column-major slices): every row still summed in CSR order,
    so a sequential-dot solve is bitwise the reference's (incl. a ragged
    last slice and window)."""
    monkeypatch.setenv("PIPECG_B200_SELL", "1")
    A = pb.generate_powerlaw(n) if n == 2**12 else _random_spd(n, 30, seed=4)
    assert A.row_nnz().max() <= 256
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                             options=pb.DeviceOptions(dot_mode="seq", engine=engine))
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)


def _hub_spd(n, hub_rows, hub_len, seed):
    """Symmetric, strictly diagonally dominant; `hub_rows` rows coupled to
    `hub_len` random columns each (rows of > 2,048 nonzeros: several chunks
    of the engine-2 long-row path, like the 49,349-nonzero rows of the
    2^22 power-law config), plus a sparse random background."""
    rng = np.random.default_rng(seed)
    r = [np.repeat(np.arange(hub_rows), hub_len)]
    c = [rng.integers(0, n, size=hub_rows * hub_len)]
    bg = rng.integers(0, n, size=(2, 4 * n))
    r.append(bg[0])
    c.append(bg[1])
    r, c = np.concatenate(r), np.concatenate(c)
    keep = r != c
    key = np.unique(np.minimum(r[keep], c[keep]) * n + np.maximum(r[keep], c[keep]))
    a, b = key // n, key % n
    v = -rng.uniform(0.1, 1.0, size=a.size)
    rows = np.concatenate([a, b, np.arange(n)])
    cols = np.concatenate([b, a, np.arange(n)])
    vals = np.concatenate([v, v, np.zeros(n)])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    vals[rows == cols] = np.bincount(rows, weights=np.abs(vals), minlength=n) + 1.0
    ro = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ro[1:])
    return pb.CsrMatrix(n, n, ro, cols, vals)


@pytest.mark.parametrize("engine", ["two", "fused-g"])
@pytest.mark.parametrize("chunk_nnz", [None, 300, 64])
def test_hub_rows_multi_chunk(cuda, monkeypatch, chunk_nnz, engine):
    """Engine 2's long-row path with several chunks per row (kChunkNnz =
    2,048 by default; PIPECG_B200_CHUNK_NNZ shrinks it so every row > 256
    nonzeros splits into many chunks): the last chunk to finish (atomic
    ticket) sums the chunk partials in chunk order.  Within the oracle's
    reorder envelope in both dot modes, and bitwise repeatable."""
    if chunk_nnz:
        monkeypatch.setenv("PIPECG_B200_CHUNK_NNZ", str(chunk_nnz))
    A = _hub_spd(60000, 6, 9000, seed=11)
    lens = A.row_nnz()
    assert lens.max() > 4 * 2048  # >= 5 chunks per hub row at the default size
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    env = envelope(A, b, x0, d, tol, 3000)
    for mode in ("tree", "seq"):
        opts = pb.DeviceOptions(engine=engine, dot_mode=mode)
        x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg, options=opts)
        assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x, env)
        x2, rep2 = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg, options=opts)
        assert rep2.history == rep.history
        np.testing.assert_array_equal(x2, x)


def test_powerlaw_multi_chunk_small_chunks(cuda, monkeypatch):
    """Power-law 2^16 (rows up to ~1,800 nonzeros) with 64-nonzero chunks:
    every row above 256 nonzeros becomes 5..29 chunks."""
    monkeypatch.setenv("PIPECG_B200_CHUNK_NNZ", "64")
    A = pb.generate_powerlaw(2**16)
    assert A.row_nnz().max() > 20 * 64
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=2000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=2000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                             options=pb.DeviceOptions(engine="two"))
    assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x,
                           envelope(A, b, x0, d, tol, 2000))


# ---------------------------------------------------------------------------
# engine 3 ("fused-g"): one SELL kernel per iteration, hub rows inside it
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["powerlaw16", "hubs", "hubs-chunk64", "ragged"])
def test_fused_g_matches_oracle(cuda, monkeypatch, case):
    """Engine 3 in both dot modes.  Rows <= 256 nonzeros are summed by their
    SELL position's thread in CSR order (k-blocks of the window staged in
    shared memory): with no hub rows a seq-dot solve is the reference's bit
    for bit.  Hub rows (warp chunks, chunk partials combined in order) are
    graded against the oracle's reorder envelope."""
    if case == "hubs-chunk64":
        monkeypatch.setenv("PIPECG_B200_CHUNK_NNZ", "64")
    A = {"powerlaw16": lambda: pb.generate_powerlaw(2**16),
         "hubs": lambda: _hub_spd(60000, 6, 9000, seed=11),
         "hubs-chunk64": lambda: _hub_spd(20000, 4, 3000, seed=5),
         "ragged": lambda: _random_spd(70001, 30, seed=8)}[case]()
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    hubs = A.row_nnz().max() > 256
    env = envelope(A, b, x0, d, tol, 3000) if hubs else None
    for mode in ("seq", "tree"):
        x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                                 options=pb.DeviceOptions(engine="fused-g", dot_mode=mode))
        if mode == "seq" and not hubs:
            assert rep.history == ref.history
            np.testing.assert_array_equal(x, ref.x)
        else:
            assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x,
                                   env or envelope(A, b, x0, d, tol, 3000))


def test_fused_g_tree_deterministic_and_in_envelope(cuda):
    """Tree mode: block partials + hub slots summed in a fixed order by the
    last CTA -> repeated solves are bitwise identical; graded against the
    oracle's reorder envelope."""
    A = _hub_spd(60000, 6, 9000, seed=11)
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    opts = pb.DeviceOptions(engine="fused-g")
    x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg, options=opts)
    assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x,
                           envelope(A, b, x0, d, tol, 3000))
    for _ in range(2):
        x2, rep2 = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg, options=opts)
        assert rep2.history == rep.history
        np.testing.assert_array_equal(x2, x)


@pytest.mark.parametrize("engine,env", [
    ("two", {"PIPECG_B200_E2POL": "0"}), ("two", {"PIPECG_B200_E2GLD": "0"}),
    ("two", {"PIPECG_B200_E2GLD": "2"}), ("two", {"PIPECG_B200_SELL_BATCH": "2"}),
    ("fused-g", {"PIPECG_B200_G_BATCH": "4"}), ("fused-g", {"PIPECG_B200_G_MB": "6"}),
    ("fused-g", {"PIPECG_B200_G_PF": "1"}), ("fused-g", {"PIPECG_B200_G_THR": "128"})])
def test_irregular_kernel_switches_bitwise(cuda, monkeypatch, engine, env):
    """The experiment switches of the irregular engines (L2 hints, gather
    cache mode, batch depth, CTAs per SM, operand prefetch, lane-row
    threshold up to 128) change only speed: a seq-dot solve is still the
    reference's bit for bit when no row is longer than 256 nonzeros, and
    within the reorder envelope otherwise."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    A = pb.generate_powerlaw(2**13)
    mx = int(A.row_nnz().max())
    b, x0, d, tol = _problem(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=2000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=2000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                             options=pb.DeviceOptions(engine=engine, dot_mode="seq"))
    if mx <= 256:
        assert rep.history == ref.history
        np.testing.assert_array_equal(x, ref.x)
    else:  # rows > 256: the init SpMVs (and engine 2) combine them with a tree
        assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x,
                               envelope(A, b, x0, d, tol, 2000))
