"""Pin the CPU oracle (oracle/pipecg_oracle.c) to the reference's own outputs.

Every fixture under tests/golden was produced by running the reference
package (tests/golden/make_golden.py); these tests need no GPU.  Bitwise
equality is required everywhere the reference is bitwise deterministic
(kernels.py:1-7): SpMV, the sequential dot, the fused update, Jacobi and
whole solver histories.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, golden_matrix, load_golden, python_dot

META = json.loads((GOLDEN / "golden_meta.json").read_text())


@pytest.fixture(scope="module")
def K():
    return load_golden("kernels.npz")


def test_fused_update_bitwise(K):
    v = {nm: K["in_" + nm] for nm in ("z", "q", "s", "p", "x", "r", "u", "w", "m", "n")}
    out = oracle.fused_update(v, float(K["alpha"]), float(K["beta"]))
    for nm in v:
        np.testing.assert_array_equal(out[nm], K["out_" + nm], err_msg=nm)


def test_dot_bitwise(K):
    assert oracle.dot(K["dot_a"], K["dot_b"]) == float(K["dot_ab"])
    assert oracle.dot(K["dot_a"], K["dot_b"]) == python_dot(K["dot_a"], K["dot_b"])


def test_dot_blocked_differs_but_close(K):
    a, b = K["dot_a"], K["dot_b"]
    ref = float(K["dot_ab"])
    got = oracle.dot_blocked(a, b)
    assert abs(got - ref) <= 1e-12 * np.sum(np.abs(a * b))


def test_spmv_bitwise_p125(K):
    A = golden_matrix(K, "p125n6")
    np.testing.assert_array_equal(oracle.spmv(A, K["p125n6_x"]), K["p125n6_y"])


def test_spmv_bitwise_rectangular(K):
    A = golden_matrix(K, "rand")
    np.testing.assert_array_equal(oracle.spmv(A, K["rand_x"]), K["rand_y"])


def test_jacobi_bitwise(K):
    A = golden_matrix(K, "p125n6")
    d = oracle.jacobi_inv_diag(A)
    np.testing.assert_array_equal(d, K["p125n6_inv_diag"])
    np.testing.assert_array_equal(oracle.jacobi_apply(d, K["p125n6_x"]), K["p125n6_jacobi"])


@pytest.mark.parametrize("key,kind,n", [("2d5_33", "2d5", 33), ("3d7_11", "3d7", 11),
                                        ("3d27_9", "3d27", 9), ("p125_7", "p125", 7)])
def test_stencil_generators_match_reference_structure(key, kind, n):
    A = oracle.stencil(kind, n)
    meta = META["stencils"][key]
    assert (A.n_rows, A.nnz) == (meta["N"], meta["nnz"])
    import hashlib

    h = hashlib.sha256()
    for arr in (A.row_offsets, A.col_indices, A.values):
        h.update(np.ascontiguousarray(arr).tobytes())
    assert h.hexdigest() == meta["sha256"]


def test_pipecg_scalars_known_answers():
    # reference tests/test_solvers.py:101-125
    assert oracle.pipecg_scalars(0.5, 123.0, 0.25, 456.0, 0) == (2.0, 0.0)
    assert oracle.pipecg_scalars(1.0, 2.0, 3.0, 0.5, 1) == (0.5, 0.5)
    assert oracle.pipecg_scalars(1.0, 1.0, 0.0, 1.0, 0)[0] == "breakdown"
    assert oracle.pipecg_scalars(1.0, 1.0, 1.0, 1.0, 3)[0] == "breakdown"
    assert oracle.pipecg_scalars(1.0, 1.0, np.inf, 1.0, 0)[0] == "breakdown"


SOLVE_CASES = [c for c in META["cases"] if c != "p125n6_pcg"]


@pytest.mark.parametrize("case", SOLVE_CASES)
def test_pipecg_solve_bitwise_history(case):
    g = load_golden(f"solve_{case}.npz")
    m = META["cases"][case]
    A = golden_matrix(g)
    res = oracle.pipecg_solve(A, g["b"], g["x0"], g["inv_diag"], tol=float(g["tol"]),
                              max_iterations=int(g["max_iterations"]),
                              record_history=True,
                              drift_check_interval=int(g["drift_k"]))
    if "breakdown" in m:
        assert res.breakdown is not None
        assert res.breakdown[0] == m["breakdown"]
        assert res.breakdown[1] == m["iteration"]
        return
    assert res.breakdown is None
    assert res.iterations == m["iterations"]
    assert res.converged == m["converged"]
    assert res.final_norm == m["final_norm"]
    np.testing.assert_array_equal(np.array(res.history), g["history"])
    np.testing.assert_array_equal(res.x, g["x"])
    if int(g["drift_k"]) > 0:
        np.testing.assert_array_equal(np.array(res.drift_history), g["drift"])


def test_pcg_solve_bitwise_history():
    g = load_golden("solve_p125n6_pcg.npz")
    m = META["cases"]["p125n6_pcg"]
    res = oracle.pcg_solve(golden_matrix(g), g["b"], g["x0"], g["inv_diag"],
                           tol=float(g["tol"]), max_iterations=int(g["max_iterations"]))
    assert res.iterations == m["iterations"]
    np.testing.assert_array_equal(np.array(res.history), g["history"])
    np.testing.assert_array_equal(res.x, g["x"])


def test_config1_2d5_512_bitwise():
    """BASELINE config 1 (2D 5-pt 512^2): the whole 894-iteration history."""
    g = load_golden("config1_2d5_512.npz")
    A = oracle.stencil("2d5", 512)
    _, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    assert tol == float(g["tol"])
    res = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    assert res.iterations == META["config1"]["iterations"] == 894
    np.testing.assert_array_equal(np.array(res.history), g["history"])
    np.testing.assert_array_equal(res.x, g["x"])


def test_reorder_envelope_small():
    """Dot reordering alone keeps the iteration count and h0-normalised gap tiny
    (SURVEY.md §8(c) noise floor) -- the yardstick for the GPU's tree dots."""
    A = oracle.stencil("3d7", 16)
    _, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    r1 = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    r2 = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000, dot_mode="blocked")
    assert r1.iterations == r2.iterations
    assert oracle.history_gap(r2.history, r1.history) <= 1e-12


def test_threaded_baseline_same_iterations():
    A = oracle.stencil("3d7", 20)
    _, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    r1 = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    try:
        oracle.set_threads(4)
        r4 = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    finally:
        oracle.set_threads(1)
    assert abs(r1.iterations - r4.iterations) <= 1
    assert np.max(np.abs(r1.x - r4.x)) <= 1e-8 * np.max(np.abs(r1.x))


@pytest.mark.parametrize("kind,n,expect", [("2d5", 10, 9), ("3d7", 6, 27), ("3d27", 5, 27),
                                           ("3d7", 2, 8), ("p125", 6, 125)])
def test_row_pattern_checker(kind, n, expect):
    """oracle.row_patterns (the checker of csrc/patterns.cu): the boundary
    classes of each stencil, codes by first occurrence, and every row
    rebuilt from its dictionary entry is the CSR row bit for bit.  p125:
    125 classes x up to 125 entries = 6,859 entries (<= 8,192)."""
    if kind == "p125":
        assert oracle.row_patterns(oracle.stencil(kind, n), max_entries=6858)[0] == 0
    A = oracle.stencil(kind, n)
    n_pat, n_e, codes = oracle.row_patterns(A)
    assert n_pat == expect
    if not expect:
        assert codes is None
        return
    ro, ci, va = A.row_offsets, A.col_indices, A.values
    first = {}
    for i in range(A.n_rows):
        first.setdefault(int(codes[i]), i)
    assert list(first) == list(range(n_pat))  # numbered by first occurrence
    assert n_e == sum(int(ro[i + 1] - ro[i]) for i in first.values())
    for i in range(A.n_rows):
        r = first[int(codes[i])]
        np.testing.assert_array_equal(ci[ro[i]:ro[i + 1]] - i, ci[ro[r]:ro[r + 1]] - r)
        np.testing.assert_array_equal(va[ro[i]:ro[i + 1]].view(np.int64),
                                      va[ro[r]:ro[r + 1]].view(np.int64))
