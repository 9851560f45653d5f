"""Fused variants E/F: the matrix read through its lossless row-pattern
dictionary (csrc/patterns.cu) instead of the CSR.

* The device dictionary equals the oracle's (oracle.row_patterns): same
  number of lists, same entries, same code for every row.
* With dot_mode="seq" every solve is bitwise the reference's: each row's
  sum runs over the same (column, value) pairs in CSR order
  (kernels.py:64-70, solvers.py:324-387).
* Matrices without a dictionary (too many distinct rows / entries) keep
  the CSR variants; asking for E/F on them fails loudly.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, golden_matrix, load_golden

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_2105_06176_b200")
torch = pytest.importorskip("torch")
from test_gpu_irregular import _random_spd  # noqa: E402
from test_gpu_solver import _rp64, assert_within_envelope, envelope  # noqa: E402

META = json.loads((GOLDEN / "golden_meta.json").read_text())
CASES = [c for c in META["cases"] if c != "p125n6_pcg"]


def _perturbed(kind, n, rows):
    """A stencil whose listed rows get a different diagonal (extra patterns)."""
    A = pb.stencil_host(kind, n)
    va = np.array(A.values, dtype=np.float64)
    ro, ci = np.asarray(A.row_offsets), np.asarray(A.col_indices)
    for i in rows:
        for k in range(ro[i], ro[i + 1]):
            if ci[k] == i:
                va[k] += 0.5 + 0.25 * (i % 3)
    return pb.CsrMatrix(A.n_rows, A.n_cols, ro, ci, va)


DICT_CASES = [("2d5", 20), ("3d7", 12), ("3d27", 9), ("3d7", 3), ("p125", 9)]


@pytest.mark.parametrize("kind,n", DICT_CASES)
def test_dictionary_matches_oracle(cuda, kind, n):
    A = pb.stencil_host(kind, n)
    n_pat, n_e, codes = pb.as_device_csr(A).row_patterns(codes=True)
    r_pat, r_e, r_codes = oracle.row_patterns(A)
    assert (n_pat, n_e) == (r_pat, r_e)
    assert n_pat == {"2d5": 9, "p125": 125}.get(kind, 27)
    if kind == "p125":
        assert n_e == 6859  # (3 + 4 + 5 + 4 + 3)^3 entries, <= the 8192 limit
    np.testing.assert_array_equal(codes.cpu().numpy(), r_codes)


def test_dictionary_perturbed_rows_and_rp64(cuda):
    A = _perturbed("3d7", 10, [0, 17, 555, 999])
    for D in (pb.as_device_csr(A), _rp64(A)):
        n_pat, n_e, codes = D.row_patterns(codes=True)
        r_pat, r_e, r_codes = oracle.row_patterns(A)
        assert (n_pat, n_e) == (r_pat, r_e) and n_pat > 27
        np.testing.assert_array_equal(codes.cpu().numpy(), r_codes)


def _wide_band(n=2000, half=40, kinds=100):
    """Band matrix (not symmetric -- never solved) whose interior rows come
    in `kinds` value sets: <= 256 row patterns but > 8,192 dictionary
    entries."""
    rows, cols, vals = [], [], []
    for i in range(n):
        for d in range(-half, half + 1):
            j = i + d
            if 0 <= j < n:
                rows.append(i)
                cols.append(j)
                vals.append(4.0 * half if d == 0 else -1.0 - (i % kinds) / 1000.0)
    ro = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ro, np.asarray(rows) + 1, 1)
    return pb.CsrMatrix(n, n, np.cumsum(ro), np.asarray(cols, dtype=np.int64), np.asarray(vals))


@pytest.mark.parametrize("make", [_wide_band, lambda: _random_spd(3000, 12, 5)])
def test_no_dictionary_when_rows_are_diverse(cuda, make):
    A = make()
    assert oracle.row_patterns(A)[0] == 0
    assert pb.as_device_csr(A).row_patterns() == (0, 0)
    b = np.ones(A.n_rows)
    with pytest.raises(Exception, match="row-pattern"):
        pb.pipecg_solve(A, b, np.zeros(A.n_rows), pb.jacobi_setup(A),
                        pb.SolverConfig(tolerance=1e-8, max_iterations=10),
                        options=pb.DeviceOptions(engine="fused-e"))


def _seq_vs_oracle(A, engine, max_it=5000, device_matrix=None):
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=max_it)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=max_it, record_history=True)
    opts = pb.DeviceOptions(dot_mode="seq", engine=engine)
    if device_matrix is None:
        x, rep = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, options=opts)
    else:
        bd = torch.from_numpy(b).cuda()
        x, rep = pb.pipecg_solve(device_matrix, bd, torch.zeros_like(bd),
                                 pb.JacobiPreconditioner(d), cfg, options=opts)
        x = x.cpu().numpy()
    assert rep.iterations == ref.iterations
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)
    return rep


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
@pytest.mark.parametrize("kind,n", [("2d5", 40), ("3d7", 20), ("3d27", 12), ("3d7", 13), ("3d7", 2),
                                    # 125 row patterns / 6,859 entries; 25 lines of
                                    # offsets bridged into 5 plane windows
                                    ("p125", 40)])
def test_stencil_seq_bitwise(cuda, kind, n, engine):
    _seq_vs_oracle(pb.stencil_host(kind, n), engine)


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
def test_perturbed_and_rp64_seq_bitwise(cuda, engine):
    A = _perturbed("3d7", 14, [3, 100, 2000, 2743])
    _seq_vs_oracle(A, engine)
    _seq_vs_oracle(A, engine, device_matrix=_rp64(A))


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
@pytest.mark.parametrize("case", CASES)
def test_golden_cases_seq_bitwise(cuda, case, engine):
    """Every golden case whose matrix has a dictionary, bit for bit."""
    g = load_golden(f"solve_{case}.npz")
    m = META["cases"][case]
    A = golden_matrix(g)
    if oracle.row_patterns(A)[0] == 0:
        pytest.skip("no row-pattern dictionary for this matrix")
    pc = pb.JacobiPreconditioner(g["inv_diag"])
    cfg = pb.SolverConfig(tolerance=float(g["tol"]), max_iterations=int(g["max_iterations"]),
                          record_history="breakdown" not in m,
                          drift_check_interval=int(g["drift_k"]))
    opts = pb.DeviceOptions(dot_mode="seq", engine=engine)
    if "breakdown" in m:
        with pytest.raises(pb.SolverBreakdown) as exc:
            pb.pipecg_solve(A, g["b"], g["x0"], pc, cfg, options=opts)
        assert exc.value.quantity == m["breakdown"]
        assert exc.value.iteration == m["iteration"]
        return
    x, rep = pb.pipecg_solve(A, g["b"], g["x0"], pc, cfg, options=opts)
    assert rep.iterations == m["iterations"]
    np.testing.assert_array_equal(np.array(rep.history), g["history"])
    np.testing.assert_array_equal(x, g["x"])


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
def test_tree_mode_within_envelope(cuda, engine):
    A = pb.stencil_host("3d7", 24)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=5000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg,
                             options=pb.DeviceOptions(engine=engine))
    assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x,
                           envelope(A, b, x0, d, tol, 5000))


def test_autotuned_engine_bitwise(cuda):
    """>= 64K rows: the autotuner times E/F beside the CSR variants; whatever
    it picks is bitwise the reference in seq mode."""
    rep = _seq_vs_oracle(pb.stencil_host("3d7", 48), "auto", max_it=3000)
    assert rep.iterations > 10


def _seq_with_dinv(A, d, engine, opts_pc=None):
    x_true, b, x0, _ = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    pc = opts_pc if opts_pc is not None else pb.JacobiPreconditioner(d)
    x, rep = pb.pipecg_solve(A, b, x0, pc, cfg, options=pb.DeviceOptions(dot_mode="seq", engine=engine))
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
def test_dinv_not_a_function_of_the_code(cuda, engine):
    """A preconditioner that is not 1/diag of the pattern (some rows scaled):
    E falls back to per-nonzero gathers, F stages dinv -- still bitwise."""
    A = pb.stencil_host("3d7", 14)
    d = oracle.jacobi_inv_diag(A).copy()
    d[[5, 77, 1000]] *= 1.0 + 2.0**-20
    _seq_with_dinv(A, d, engine)


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
def test_dinv_changed_in_place_between_solves(cuda, engine):
    """The cached solver re-checks dinv at every solve (solver_init)."""
    A = pb.stencil_host("3d7", 12)
    d0 = oracle.jacobi_inv_diag(A)
    dev = torch.from_numpy(d0.copy()).cuda()
    pc = pb.JacobiPreconditioner(dev)
    _seq_with_dinv(A, d0, engine, pc)
    d1 = d0.copy()
    d1[[3, 500]] *= 1.0 - 2.0**-18
    dev.copy_(torch.from_numpy(d1))
    _seq_with_dinv(A, d1, engine, pc)
    dev.copy_(torch.from_numpy(d0))
    _seq_with_dinv(A, d0, engine, pc)


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
@pytest.mark.parametrize("max_it", [1, 2, 3, 10, 11])
def test_deferred_x_every_stop_parity(cuda, engine, max_it):
    """E/F update x every other iteration (both updates, in order, on odd
    iterations; the stopping kernel applies a pending one): x after a stop at
    either parity -- max_iterations or convergence -- is bitwise the reference's."""
    A = pb.stencil_host("3d7", 16)
    x_true, b, x0, d = oracle.manufactured(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=1e-300, max_iterations=max_it)
    cfg = pb.SolverConfig(tolerance=1e-300, max_iterations=max_it, record_history=True)
    for chunk in (0, 3):
        x, rep = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg,
                                 options=pb.DeviceOptions(dot_mode="seq", engine=engine,
                                                          chunk=chunk))
        assert rep.iterations == max_it
        np.testing.assert_array_equal(x, ref.x)


@pytest.mark.parametrize("engine", ["fused-e", "fused-f"])
def test_drift_samples_with_row_patterns(cuda, engine):
    """Drift samples read x: E/F then update x every iteration; the cached
    solver switches between the two modes across solves."""
    A = pb.stencil_host("3d7", 14)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000, drift_check_interval=5)
    pc = pb.JacobiPreconditioner(d)
    opts = pb.DeviceOptions(dot_mode="seq", engine=engine)
    for k in (0, 5, 0):
        cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True,
                              drift_check_interval=k)
        x, rep = pb.pipecg_solve(A, b, x0, pc, cfg, options=opts)
        np.testing.assert_array_equal(x, ref.x)
        if k:
            assert [t[0] for t in rep.drift_history] == [t[0] for t in ref.drift_history]


def _nine_point(n):
    """2D 9-point Laplacian-like SPD matrix (diag 8, 8 neighbours -1),
    assembled here: a stencil the generators do not produce."""
    rows, cols, vals = [], [], []
    for y in range(n):
        for x in range(n):
            i = y * n + x
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    xx, yy = x + dx, y + dy
                    if 0 <= xx < n and 0 <= yy < n:
                        rows.append(i)
                        cols.append(yy * n + xx)
                        vals.append(8.0 if (dx, dy) == (0, 0) else -1.0)
    ro = np.zeros(n * n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n * n), out=ro[1:])
    return pb.CsrMatrix(n * n, n * n, ro, np.array(cols, dtype=np.int64), np.array(vals))


def _tridiag(n):
    ro = np.zeros(n + 1, dtype=np.int64)
    cols, vals = [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                cols.append(j)
                vals.append(2.5 if j == i else -1.0)
        ro[i + 1] = len(cols)
    return pb.CsrMatrix(n, n, ro, np.array(cols, dtype=np.int64), np.array(vals))


@pytest.mark.parametrize("engine", ["fused-e", "fused-f", "auto"])
@pytest.mark.parametrize("make", [lambda: _nine_point(45), lambda: _tridiag(37),
                                  lambda: _tridiag(300000)])
def test_assembled_matrices_seq_bitwise(cuda, make, engine):
    """Matrices assembled outside the generators (9-point 2D, tridiagonal
    with n not a multiple of any tile height, one with >= 64K rows so the
    autotuner runs): dictionary = oracle's, solves bitwise."""
    A = make()
    n_pat, n_e = pb.as_device_csr(A).row_patterns()
    assert (n_pat, n_e) == oracle.row_patterns(A)[:2]
    _seq_vs_oracle(A, engine, max_it=400)


@pytest.mark.parametrize("max_sms", [0, 64, 20])
def test_autotune_alternatives_fit_the_partials(cuda, max_sms):
    """Regression: an autotune alternative (F at 128-row tiles, 6 CTAs/SM)
    launched a larger grid than any variant's default plan and wrote its
    block partials past the buffer (illegal access with max_sms=64).  The
    autotuned solve must run and stay bitwise in seq mode."""
    A = pb.stencil_host("3d7", 48)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    for dot_mode in ("seq", "tree"):
        opts = pb.DeviceOptions(dot_mode=dot_mode, engine="auto", max_sms=max_sms)
        x, rep = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, options=opts)
        if dot_mode == "seq":
            assert rep.history == ref.history
            np.testing.assert_array_equal(x, ref.x)
        else:
            assert abs(rep.iterations - ref.iterations) <= 1


def test_in_place_edits_of_cached_host_arrays_are_seen(cuda):
    """ADVICE/VERDICT r1: the device copies cached on a host CsrMatrix /
    JacobiPreconditioner must not go stale when the caller rewrites the
    arrays in place (the reference reads them afresh every call).  Scale
    the matrix values and the preconditioner in place between two solves:
    the second solve is the oracle's solve of the edited system."""
    A = pb.stencil_host("3d7", 16)
    pc = pb.jacobi_setup(A)
    x_true, b, x0, d = oracle.manufactured(A)
    cfg = pb.SolverConfig(tolerance=1e-10, max_iterations=2000, record_history=True)
    opts = pb.DeviceOptions(dot_mode="seq")
    pb.pipecg_solve(A, b, x0, pc, cfg, options=opts)  # caches the device copies
    A.values[:] *= 3.0          # in place: same arrays, new content
    pc.inv_diag[:] /= 3.0
    ref = oracle.pipecg_solve(A, b, x0, pc.inv_diag, tol=1e-10, max_iterations=2000)
    x, rep = pb.pipecg_solve(A, b, x0, pc, cfg, options=opts)
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)
