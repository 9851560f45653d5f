"""GPU parity of pipecg_solve against the reference's goldens and the oracle.

Gates (BASELINE.md "Parity gates"):
  1. iteration count within +-1 of the oracle,
  2. G = max_k |h_k - h_k^ref| / h_0 <= max(1e-10, 3E)  (E: dot-reorder envelope),
  3. final x within 1e-8 relative,
  4. dot_mode="seq": history and x bitwise identical to the reference.
"""

from __future__ import annotations

import json
import math

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, golden_matrix, load_golden

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_2105_06176_b200")
torch = pytest.importorskip("torch")

META = json.loads((GOLDEN / "golden_meta.json").read_text())
SEQ = pb.DeviceOptions(dot_mode="seq")


def _cfg(g, record=True):
    return pb.SolverConfig(tolerance=float(g["tol"]), max_iterations=int(g["max_iterations"]),
                           record_history=record, drift_check_interval=int(g["drift_k"]))


CASES = [c for c in META["cases"] if c != "p125n6_pcg"]


@pytest.mark.parametrize("engine", ["fused-a", "fused-b", "fused-c", "fused-d", "fused-p", "two"])
@pytest.mark.parametrize("case", CASES)
def test_golden_bitwise_seq_mode(cuda, case, engine):
    """dot_mode='seq' reproduces the reference solve bit for bit."""
    g = load_golden(f"solve_{case}.npz")
    m = META["cases"][case]
    A = golden_matrix(g)
    pc = pb.JacobiPreconditioner(g["inv_diag"])
    opts = pb.DeviceOptions(dot_mode="seq", engine=engine)
    if "breakdown" in m:
        with pytest.raises(pb.SolverBreakdown) as exc:
            pb.pipecg_solve(A, g["b"], g["x0"], pc, _cfg(g, False), options=opts)
        assert exc.value.quantity == m["breakdown"]
        assert exc.value.iteration == m["iteration"]
        return
    x, rep = pb.pipecg_solve(A, g["b"], g["x0"], pc, _cfg(g), options=opts)
    assert rep.iterations == m["iterations"]
    assert rep.converged == m["converged"]
    assert rep.final_norm == m["final_norm"]
    assert rep.strategy == "pipecg"
    np.testing.assert_array_equal(np.array(rep.history), g["history"])
    np.testing.assert_array_equal(x, g["x"])
    if int(g["drift_k"]) > 0:
        assert [d[0] for d in rep.drift_history] == [int(d) for d in g["drift"][:, 0]]
        np.testing.assert_allclose(np.array(rep.drift_history)[:, 1], g["drift"][:, 1],
                                   rtol=1e-6, atol=1e-15)


def envelope(A, b, x0, d, tol, max_iterations, drift_k=0):
    """The oracle's own parity noise floor at this config: the reference
    algorithm with only its dot order changed (256 sequential partials +
    pairwise tree).  Returns (iteration gap, h0-normalised history gap E,
    x relative gap) between the two oracle runs (BASELINE.md gate 2)."""
    r1 = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=max_iterations)
    r2 = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=max_iterations,
                             dot_mode="blocked")
    scale = max(np.max(np.abs(r1.x)), 1e-300)
    return (abs(r1.iterations - r2.iterations), oracle.history_gap(r2.history, r1.history),
            float(np.max(np.abs(r1.x - r2.x)) / scale))


def assert_within_envelope(x, rep, ref_iters, ref_hist, ref_x, env):
    it_gap, E, x_gap = env
    assert abs(rep.iterations - ref_iters) <= max(1, it_gap), (rep.iterations, ref_iters, env)
    G = oracle.history_gap(rep.history, list(ref_hist))
    assert G <= max(1e-10, 3 * E), (G, env)
    scale = max(np.max(np.abs(ref_x)), 1e-300)
    rel = float(np.max(np.abs(x - ref_x)) / scale)
    assert rel <= max(1e-8, 3 * x_gap), (rel, env)


@pytest.mark.parametrize("engine", ["fused-a", "fused-b", "fused-c", "fused-d", "fused-p", "two"])
@pytest.mark.parametrize("case", CASES)
def test_golden_tree_mode_tolerance(cuda, case, engine):
    """Default (tree dots): iterations, history and x within the larger of the
    BASELINE.md gates (+-1, 1e-10, 1e-8) and 3x the oracle's reorder envelope."""
    g = load_golden(f"solve_{case}.npz")
    m = META["cases"][case]
    A = golden_matrix(g)
    pc = pb.JacobiPreconditioner(g["inv_diag"])
    opts = pb.DeviceOptions(engine=engine)
    if "breakdown" in m:
        with pytest.raises(pb.SolverBreakdown) as exc:
            pb.pipecg_solve(A, g["b"], g["x0"], pc, _cfg(g, False), options=opts)
        assert exc.value.quantity == m["breakdown"]
        return
    x, rep = pb.pipecg_solve(A, g["b"], g["x0"], pc, _cfg(g), options=opts)
    env = envelope(A, g["b"], g["x0"], g["inv_diag"], float(g["tol"]), int(g["max_iterations"]))
    assert_within_envelope(x, rep, m["iterations"], g["history"], g["x"], env)


def test_config1_2d5_512_parity(cuda):
    """BASELINE config 1 vs the reference's own 894-iteration run."""
    g = load_golden("config1_2d5_512.npz")
    A = pb.stencil_host("2d5", 512)
    x_true = np.full(A.n_rows, 1.0 / math.sqrt(A.n_rows))
    b = pb.spmv(A, x_true)
    pc = pb.jacobi_setup(A)
    tol = float(g["tol"])
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, np.zeros(A.n_rows), pc, cfg)
    assert abs(rep.iterations - 894) <= 1
    G = oracle.history_gap(rep.history, list(g["history"]))
    assert G <= max(1e-10, 3 * 3.0e-12), G
    rel = np.max(np.abs(x - g["x"])) / np.max(np.abs(g["x"]))
    assert rel <= 1e-8, rel
    # bitwise mode on the same config
    x2, rep2 = pb.pipecg_solve(A, b, np.zeros(A.n_rows), pc, cfg, options=SEQ)
    assert rep2.iterations == 894
    np.testing.assert_array_equal(np.array(rep2.history), g["history"])
    np.testing.assert_array_equal(x2, g["x"])


@pytest.mark.parametrize("kind,n", [("3d7", 32), ("3d27", 20), ("p125", 12), ("2d5", 100)])
def test_stencils_vs_oracle(cuda, kind, n):
    A = pb.stencil_host(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    pc = pb.jacobi_setup(A)
    np.testing.assert_array_equal(pc.inv_diag, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pc, cfg)
    env = envelope(A, b, x0, d, tol, 20000)
    assert_within_envelope(x, rep, ref.iterations, ref.history, ref.x, env)
    xs, reps = pb.pipecg_solve(A, b, x0, pc, cfg, options=SEQ)
    assert reps.history == ref.history
    np.testing.assert_array_equal(xs, ref.x)


def test_determinism_bitwise(cuda):
    """Acceptance #10 (test_acceptance.py:328-358): repeated runs identical."""
    A = pb.stencil_host("3d7", 40)
    x_true = np.full(A.n_rows, 1 / math.sqrt(A.n_rows))
    b = pb.spmv(A, x_true)
    pc = pb.jacobi_setup(A)
    cfg = pb.SolverConfig(tolerance=1e-9, record_history=True)
    x1, r1 = pb.pipecg_solve(A, b, np.zeros(A.n_rows), pc, cfg)
    x2, r2 = pb.pipecg_solve(A, b, np.zeros(A.n_rows), pc, cfg)
    assert r1.history == r2.history
    np.testing.assert_array_equal(x1, x2)


def test_device_tensor_inputs(cuda):
    Ad = pb.stencil_device("3d7", 30)
    n = Ad.n_rows
    x_true = torch.full((n,), 1 / math.sqrt(n), dtype=torch.float64, device="cuda")
    b = pb.spmv(Ad, x_true)
    pc = pb.jacobi_setup(Ad)
    x, rep = pb.pipecg_solve(Ad, b, torch.zeros_like(b), pc, pb.SolverConfig(tolerance=1e-10))
    assert isinstance(x, torch.Tensor) and x.is_cuda
    assert rep.converged
    assert float((x - x_true).abs().max()) < 1e-7


def test_max_iterations_and_chunk_boundaries(cuda):
    A = pb.stencil_host("3d7", 16)
    x_true, b, x0, d = oracle.manufactured(A)
    pc = pb.JacobiPreconditioner(d)
    for maxit in (1, 2, 3, 4, 5, 7, 8, 9, 31, 64):
        for chunk in (4, 8, 16):
            cfg = pb.SolverConfig(max_iterations=maxit, tolerance=1e-300, record_history=True)
            x, rep = pb.pipecg_solve(A, b, x0, pc, cfg,
                                     options=pb.DeviceOptions(dot_mode="seq", chunk=chunk))
            ref = oracle.pipecg_solve(A, b, x0, d, tol=1e-300, max_iterations=maxit)
            assert rep.iterations == maxit == ref.iterations
            assert not rep.converged
            assert rep.history == ref.history
            np.testing.assert_array_equal(x, ref.x)


def test_no_graphs_path(cuda):
    A = pb.stencil_host("2d5", 40)
    x_true, b, x0, d = oracle.manufactured(A)
    pc = pb.JacobiPreconditioner(d)
    cfg = pb.SolverConfig(tolerance=1e-9, record_history=True)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=1e-9)
    x, rep = pb.pipecg_solve(A, b, x0, pc, cfg,
                             options=pb.DeviceOptions(dot_mode="seq", use_graphs=False))
    assert rep.history == ref.history


def test_host_abi_solve(cuda):
    """pipecg_b200_solve_host: the one-call C-ABI drop-in with host buffers."""
    import ctypes

    from paper_2105_06176_b200 import _lib

    A = oracle.stencil("3d7", 20)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=5000)
    x = np.empty(A.n_rows)
    hist = np.empty(5001)
    res = _lib.PcgResult()
    P = lambda a, t=ctypes.c_double: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
    _lib.call("pipecg_b200_solve_host", A.n_rows, P(A.row_offsets, ctypes.c_int64),
              P(A.col_indices, ctypes.c_int64), P(A.values), P(b), P(x0), P(d), tol, 5000, 0,
              _lib.PCG_DOT_SEQ, P(x), P(hist), hist.size, None, None, 0, ctypes.byref(res))
    assert res.status == _lib.PCG_STOPPED and res.converged
    assert res.iterations == ref.iterations
    np.testing.assert_array_equal(hist[: res.n_history], np.array(ref.history))
    np.testing.assert_array_equal(x, ref.x)


def test_pipecg_init_matches_operators(cuda):
    # reference tests/test_solvers.py:153-170
    K = load_golden("kernels.npz")
    dense = np.zeros((5, 5))
    for i, cols in enumerate(((0, 1, 3), (0, 1, 4), (2, 3), (0, 2, 3, 4), (1, 3, 4))):
        for j in cols:
            dense[i, j] = 4.0 if i == j else -1.0
    A = pb.csr_from_dense(dense)
    rng = np.random.default_rng(31)
    b = rng.standard_normal(5)
    x0 = rng.standard_normal(5)
    pc = pb.jacobi_setup(A)
    st = pb.pipecg_init(A, b, x0, pc)
    r = b - pb.spmv(A, x0)
    u = pb.jacobi_apply(pc, r)
    w = pb.spmv(A, u)
    np.testing.assert_array_equal(st.r, r)
    np.testing.assert_array_equal(st.u, u)
    np.testing.assert_array_equal(st.w, w)
    np.testing.assert_array_equal(st.m, pb.jacobi_apply(pc, w))
    np.testing.assert_array_equal(st.n, pb.spmv(A, pb.jacobi_apply(pc, w)))
    assert st.gamma == pb.dot(r, u)
    assert st.delta == pb.dot(w, u)
    assert st.norm == math.sqrt(pb.dot(u, u))
    for nm in ("z", "q", "s", "p"):
        np.testing.assert_array_equal(getattr(st, nm), np.zeros(5))
    del K


@pytest.mark.parametrize("kind,n,maxit,tol", [("2d5", 64, 20000, None), ("3d7", 24, 37, None),
                                              ("3d7", 24, 20000, 1e-300), ("2d5", 300, 20000, None)])
def test_persistent_chunks_bitwise_equal_per_iteration_launches(cuda, kind, n, maxit, tol):
    """Variant P (a whole chunk of iterations in one cooperative launch,
    grid barrier between iterations) computes exactly what C computes with
    one launch per iteration: identical history and x, including stops in
    the middle of a chunk (convergence, max_iterations)."""
    A = pb.stencil_host(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = tol or oracle.recipe_tolerance(A, b, d)
    pc = pb.JacobiPreconditioner(d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=maxit, record_history=True)
    runs = {}
    for eng, chunk in (("fused-c", 8), ("fused-p", 16), ("fused-p", 7), ("fused-p", 0)):
        runs[(eng, chunk)] = pb.pipecg_solve(A, b, x0, pc, cfg,
                                             options=pb.DeviceOptions(engine=eng, chunk=chunk))
    xc, rc = runs[("fused-c", 8)]
    for key, (x, rep) in runs.items():
        assert rep.iterations == rc.iterations, key
        assert rep.history == rc.history, key
        np.testing.assert_array_equal(x, xc)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=maxit)
    assert abs(rc.iterations - ref.iterations) <= 1


def test_persistent_chunks_breakdown_mid_chunk(cuda):
    g = load_golden("solve_indefinite.npz")
    A = golden_matrix(g)
    opts = pb.DeviceOptions(engine="fused-p", chunk=16)
    with pytest.raises(pb.SolverBreakdown) as exc:
        pb.pipecg_solve(A, g["b"], g["x0"], pb.JacobiPreconditioner(g["inv_diag"]),
                        _cfg(g, False), options=opts)
    assert exc.value.quantity == "alpha denominator"


def _rp64(A):
    """The same device matrix with int64 row pointers (the layout shards with
    >= 2^31 nonzeros use), to run the long-long instantiations at small size."""
    d = pb.as_device_csr(A)
    rp = torch.empty(d.rowptr.numel(), dtype=torch.int64, device=d.rowptr.device)
    rp.copy_(d.rowptr.to(torch.int64))
    return pb.DeviceCsr(d.n_rows, d.n_cols, d.nnz, rp, d.col, d.val)


@pytest.mark.parametrize("engine", ["fused-a", "fused-b", "fused-c", "fused-d", "fused-p", "two"])
def test_int64_row_pointers_bitwise(cuda, engine):
    A = pb.stencil_host("3d7", 20)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=5000)
    D = _rp64(A)
    assert D.rp64 == 1
    bd = torch.from_numpy(b).cuda()
    np.testing.assert_array_equal(pb.spmv(D, torch.from_numpy(x_true).cuda()).cpu().numpy(),
                                  oracle.spmv(A, x_true))
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True)
    x, rep = pb.pipecg_solve(D, bd, torch.zeros_like(bd), pb.JacobiPreconditioner(d), cfg,
                             options=pb.DeviceOptions(dot_mode="seq", engine=engine))
    assert rep.history == ref.history
    np.testing.assert_array_equal(x.cpu().numpy(), ref.x)


@pytest.mark.parametrize("engine,sell", [("fused-d", "0"), ("two", "0"), ("two", "1")])
def test_int64_row_pointers_irregular_bitwise(cuda, monkeypatch, engine, sell):
    monkeypatch.setenv("PIPECG_B200_SELL", sell)
    A = pb.generate_powerlaw(2**12)  # rows up to 205 nonzeros: no hub tiles
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=2000)
    D = _rp64(A)
    bd = torch.from_numpy(b).cuda()
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=2000, record_history=True)
    x, rep = pb.pipecg_solve(D, bd, torch.zeros_like(bd), pb.JacobiPreconditioner(d), cfg,
                             options=pb.DeviceOptions(dot_mode="seq", engine=engine))
    assert rep.history == ref.history
    np.testing.assert_array_equal(x.cpu().numpy(), ref.x)


@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_non_finite_rhs_exits_like_reference(cuda, bad):
    """solvers.py:346: a NaN norm fails `norm >= tol` and exits unconverged at
    once; an inf norm keeps iterating until the recurrence breaks down --
    whatever the oracle does, the GPU must do the same."""
    A = pb.stencil_host("2d5", 20)
    x_true, b, x0, d = oracle.manufactured(A)
    b = b.copy()
    b[7] = bad
    cfg = pb.SolverConfig(tolerance=1e-8, max_iterations=50, record_history=True)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=1e-8, max_iterations=50)
    for eng in ("fused-c", "fused-p", "two"):
        opts = pb.DeviceOptions(dot_mode="seq", engine=eng)
        if ref.breakdown is not None:
            with pytest.raises(pb.SolverBreakdown) as exc:
                pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, options=opts)
            assert (exc.value.quantity, exc.value.iteration) == ref.breakdown[:2]
            continue
        x, rep = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, options=opts)
        assert rep.iterations == ref.iterations and rep.converged == ref.converged
        np.testing.assert_array_equal(np.array(rep.history), np.array(ref.history))


def test_pcg_solve_golden_bitwise_seq(cuda):
    """Classic PCG (solvers.py:195-273) on the device operators, sequential
    dots: the reference's own 5-iteration history bit for bit."""
    g = load_golden("solve_p125n6_pcg.npz")
    m = META["cases"]["p125n6_pcg"]
    A = golden_matrix(g)
    x, rep = pb.pcg_solve(A, g["b"], g["x0"], pb.JacobiPreconditioner(g["inv_diag"]),
                          _cfg(g), options=pb.DeviceOptions(dot_mode="seq"))
    assert rep.strategy == "pcg" and rep.iterations == m["iterations"]
    np.testing.assert_array_equal(np.array(rep.history), g["history"])
    np.testing.assert_array_equal(x, g["x"])


@pytest.mark.parametrize("kind,n", [("3d7", 24), ("2d5", 100)])
def test_pcg_solve_tree_vs_oracle_and_pipecg(cuda, kind, n):
    """Tree dots within the oracle's envelope; PCG and PIPECG histories agree
    over the first 20 iterations (acceptance #4, test_acceptance.py:136-154)."""
    A = pb.stencil_host(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pcg_solve(A, b, x0, d, tol=tol, max_iterations=5000)
    ref2 = oracle.pcg_solve(A, b, x0, d, tol=tol, max_iterations=5000, dot_mode="blocked")
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True)
    x, rep = pb.pcg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg)
    E = oracle.history_gap(ref2.history, ref.history)
    assert abs(rep.iterations - ref.iterations) <= 1
    assert oracle.history_gap(rep.history, ref.history) <= max(1e-10, 3 * E)
    _, rp = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg)
    h1, h2 = np.array(rep.history[:20]), np.array(rp.history[:20])
    assert np.max(np.abs(h1 - h2) / h1) <= 1e-6


def _pcg_cases():
    from test_gpu_irregular import _random_spd
    return {
        "3d7-20": lambda: pb.stencil_host("3d7", 20),
        "2d5-64": lambda: pb.stencil_host("2d5", 64),
        "powerlaw-12": lambda: pb.generate_powerlaw(2 ** 12),
        "ragged": lambda: _random_spd(3001, 20, seed=3),
    }


@pytest.mark.parametrize("case", ["3d7-20", "2d5-64", "powerlaw-12", "ragged"])
def test_pcg_device_seq_bitwise_vs_oracle(cuda, case):
    """Device PCG (engine 4: two kernels per iteration, on-device stop test,
    graph chunks) in seq-dot mode is the reference's PCG bit for bit: the
    whole history, the iteration count and x (oracle.pcg_solve restates
    solvers.py:195-273)."""
    A = _pcg_cases()[case]()
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pcg_solve(A, b, x0, d, tol=tol, max_iterations=5000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True)
    x, rep = pb.pcg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg,
                          options=pb.DeviceOptions(dot_mode="seq"))
    assert rep.strategy == "pcg" and rep.converged == ref.converged
    assert rep.iterations == ref.iterations
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)


@pytest.mark.parametrize("max_it", [1, 2, 7, 64, 65])
def test_pcg_device_budget_and_chunks(cuda, max_it):
    """max_iterations across CUDA-graph chunk boundaries: exactly max_it
    iterations, history of max_it + 1 norms, identical prefix."""
    A = pb.stencil_host("3d7", 16)
    _, b, x0, d = oracle.manufactured(A)
    ref = oracle.pcg_solve(A, b, x0, d, tol=1e-300, max_iterations=max_it)
    cfg = pb.SolverConfig(tolerance=1e-300, max_iterations=max_it, record_history=True)
    x, rep = pb.pcg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg,
                          options=pb.DeviceOptions(dot_mode="seq"))
    assert rep.iterations == max_it and not rep.converged
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)


def test_pcg_device_breakdown_matches_oracle(cuda):
    """An indefinite matrix: PCG's delta <= 0 guard (solvers.py:247-248)
    fires at the oracle's iteration with the oracle's value."""
    g = load_golden("solve_indefinite.npz")
    A = golden_matrix(g)
    b, x0, d = g["b"], g["x0"], g["inv_diag"]
    ref = oracle.pcg_solve(A, b, x0, d, tol=1e-8, max_iterations=50)
    cfg = pb.SolverConfig(tolerance=1e-8, max_iterations=50)
    if ref.breakdown is None:
        x, rep = pb.pcg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg,
                              options=pb.DeviceOptions(dot_mode="seq"))
        assert rep.iterations == ref.iterations
        return
    with pytest.raises(pb.SolverBreakdown) as exc:
        pb.pcg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg,
                     options=pb.DeviceOptions(dot_mode="seq"))
    assert (exc.value.quantity, exc.value.iteration) == ref.breakdown[:2]
    assert exc.value.value == ref.breakdown[2]


@pytest.mark.parametrize("mode", ["seq", "tree"])
def test_pcg_device_hub_rows(cuda, mode):
    """Rows longer than kLongRow (6 rows of ~9,000 nonzeros, several engine-2
    chunks each) go through pcg_hub_kernel (fixed-tree chunks, in-order
    chunk combine, the hub terms of delta summed in row order): within the
    oracle's reorder envelope in both dot modes and bitwise repeatable."""
    from test_gpu_irregular import _hub_spd

    A = _hub_spd(60000, 6, 9000, seed=11)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pcg_solve(A, b, x0, d, tol=tol, max_iterations=3000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=3000, record_history=True)
    opts = pb.DeviceOptions(dot_mode=mode)
    x, rep = pb.pcg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, options=opts)
    ref2 = oracle.pcg_solve(A, b, x0, d, tol=tol, max_iterations=3000, dot_mode="blocked")
    E = oracle.history_gap(ref2.history, ref.history)
    assert abs(rep.iterations - ref.iterations) <= max(1, abs(ref2.iterations - ref.iterations))
    assert oracle.history_gap(rep.history, ref.history) <= max(1e-10, 3 * E)
    assert np.max(np.abs(x - ref.x)) / np.max(np.abs(ref.x)) <= 1e-8
    x2, rep2 = pb.pcg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, options=opts)
    assert rep2.history == rep.history
    np.testing.assert_array_equal(x2, x)


@pytest.mark.parametrize("kind,n", [("3d7", 128), ("p125", 40)])
def test_pcg_device_config_scale_vs_oracle(cuda, kind, n):
    """Device PCG at a realistic size (3D 7-pt 128^3: 2.1M rows, ~300
    iterations; 125-point 40^3: 7.3M nonzeros): seq dots bit for bit the
    oracle's PCG (history, count, x); tree dots within the oracle's
    blocked-dot envelope (BASELINE.md gates)."""
    A = oracle.stencil(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pcg_solve(A, b, x0, d, tol=tol, max_iterations=5000)
    ref2 = oracle.pcg_solve(A, b, x0, d, tol=tol, max_iterations=5000, dot_mode="blocked")
    E = oracle.history_gap(ref2.history, ref.history)
    Ad = pb.stencil_device(kind, n)
    bd = torch.as_tensor(b, device="cuda")
    pc = pb.JacobiPreconditioner(torch.as_tensor(d, device="cuda"))
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True)
    x, rep = pb.pcg_solve(Ad, bd, torch.zeros_like(bd), pc, cfg,
                          options=pb.DeviceOptions(dot_mode="seq"))
    assert rep.iterations == ref.iterations and rep.history == ref.history
    np.testing.assert_array_equal(x.cpu().numpy(), ref.x)
    x, rep = pb.pcg_solve(Ad, bd, torch.zeros_like(bd), pc, cfg)
    assert abs(rep.iterations - ref.iterations) <= 1
    assert oracle.history_gap(rep.history, ref.history) <= max(1e-10, 3 * E)
    xs = x.cpu().numpy()
    assert np.max(np.abs(xs - ref.x)) / np.max(np.abs(ref.x)) <= max(
        1e-8, 3 * np.max(np.abs(ref2.x - ref.x)) / np.max(np.abs(ref.x)))


def test_drift_samples_config_scale(cuda):
    """Drift samples every 50 iterations on 3D 7-pt 128^3 (2.1M rows, the
    autotuned engine -- E/F then update x every iteration): the sample
    iterations are the reference's (solvers.py:371-372), every value meets
    the reference's own bound (test_solvers.py:220-230) and sits at the
    oracle's rounding-noise level, and the history passes the gates."""
    A = oracle.stencil("3d7", 128)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=5000, drift_check_interval=50)
    ref2 = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=5000, dot_mode="blocked")
    E = oracle.history_gap(ref2.history, ref.history)
    Ad = pb.stencil_device("3d7", 128)
    bd = torch.as_tensor(b, device="cuda")
    pc = pb.JacobiPreconditioner(torch.as_tensor(d, device="cuda"))
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True,
                          drift_check_interval=50)
    x, rep = pb.pipecg_solve(Ad, bd, torch.zeros_like(bd), pc, cfg)
    assert abs(rep.iterations - ref.iterations) <= 1
    assert oracle.history_gap(rep.history, ref.history) <= max(1e-10, 3 * E)
    got = [it for it, _ in rep.drift_history]
    want = [it for it, _ in ref.drift_history]
    assert got == want[: len(got)] and len(got) >= len(want) - 1
    b_norm = float(np.linalg.norm(b))
    noise = max(v for _, v in ref.drift_history)
    for it, v in rep.drift_history:
        assert 0 <= v <= 1e-10 * max(1.0, b_norm)
        assert v <= 100 * noise + 1e-15, (it, v, noise)


@pytest.mark.parametrize("engine", ["auto", "fused-e", "fused-f", "fused-a", "two"])
def test_breakdown_at_scale_matches_oracle(cuda, engine):
    """An indefinite 3D 7-pt 64^3 system (every 7th diagonal -6: Jacobi's
    u = D^-1 r then has mixed signs and gamma = (r, u) turns negative) at
    262K rows: the device raises the reference's SolverBreakdown
    (solvers.py:354-357) -- same quantity and iteration, the value bit for
    bit in seq mode and to reduction-order noise in tree mode.  The row
    classes x diagonal sign give a 46-code dictionary, so E/F run."""
    A = oracle.stencil("3d7", 64)
    n = A.n_rows
    va = np.array(A.values)
    rows = np.repeat(np.arange(n), np.diff(A.row_offsets))
    va[(A.col_indices == rows) & (rows % 7 == 0)] = -6.0
    A = pb.CsrMatrix(n, n, A.row_offsets, A.col_indices, va)
    d = oracle.jacobi_inv_diag(A)
    b = oracle.spmv(A, np.full(n, 1 / np.sqrt(n)))
    ref = oracle.pipecg_solve(A, b, np.zeros(n), d, tol=1e-12, max_iterations=3000)
    q, it, val = ref.breakdown
    cfg = pb.SolverConfig(tolerance=1e-12, max_iterations=3000)
    for mode in ("seq", "tree"):
        with pytest.raises(pb.SolverBreakdown) as e:
            pb.pipecg_solve(A, b, np.zeros(n), pb.JacobiPreconditioner(d), cfg,
                            options=pb.DeviceOptions(engine=engine, dot_mode=mode))
        assert (e.value.quantity, e.value.iteration) == (q, it)
        if mode == "seq":
            assert e.value.value == val
        else:
            assert abs(e.value.value - val) <= 1e-9 * abs(val)
