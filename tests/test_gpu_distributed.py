"""The multi-GPU device protocol on ONE B200: P "virtual ranks" in one
process (one thread + one stream + one solver each, grids sized so all
ranks are co-resident), exchanging halo rows and dot partials through the
same peer-memory exchange kernel and in-kernel waits that the multi-process
NVLink path uses (only the pointer source differs: direct vs CUDA IPC).

Parity: the sharded solve must match the single-GPU solve within the
oracle's reorder envelope (only the dot reduction order differs; every row
of the sharded SpMV is bitwise the global one)."""

from __future__ import annotations

import math
import threading

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

pb = pytest.importorskip("paper_2105_06176_b200")
torch = pytest.importorskip("torch")
from paper_2105_06176_b200 import distributed as D  # noqa: E402
from paper_2105_06176_b200._device import shared_max_sms  # noqa: E402


@pytest.fixture(autouse=True)
def _quiesce():
    """Virtual ranks share one GPU from threads of this process: a
    device-wide synchronisation in one rank's thread (a cudaFree from
    collecting an earlier test's objects, the caching allocator releasing
    blocks) while a peer's kernel spins on its arrival stalls the exchange.
    Collect and release before the ranks start (the library itself defers
    its own device-synchronising frees while connected solvers live)."""
    import gc

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    yield


def run_virtual(world, make_problem, cfg, chunk=0, engine="fused"):
    """Solve with `world` virtual ranks (threads sharing GPU 0); every rank's
    error fails the test (no retry)."""
    out, errs = _run_virtual_once(world, make_problem, cfg, chunk, engine)
    for r, e in errs:  # full messages (the assertion repr truncates them)
        print(f"rank {r}: {e}")
    assert not errs, errs
    return out


def _run_virtual_once(world, make_problem, cfg, chunk, engine):
    G = D.LocalGroup(world)
    out = [None] * world
    errs = []
    opts = pb.DeviceOptions(max_sms=shared_max_sms(world), chunk=chunk, engine=engine)

    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            prob = make_problem(g)
            xt, b = D.manufactured_local(prob)
            x, rep = D.pipecg_solve_distributed(prob, b, torch.zeros_like(b), cfg, g, opts)
            out[r] = (x.cpu().numpy(), rep, prob.plan)
        except BaseException as e:  # noqa: BLE001
            errs.append((r, repr(e)))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    return out, errs


@pytest.mark.parametrize("world,kind,n,engine", [(2, "3d7", 40, "fused-a"), (3, "3d7", 33, "fused-b"),
                                                 (2, "2d5", 200, "fused-c"), (4, "3d27", 24, "fused"),
                                                 (3, "3d27", 20, "fused-c"), (2, "3d7", 30, "fused-d"),
                                                 (2, "3d7", 40, "fused-e"), (3, "3d7", 33, "fused-f"),
                                                 (2, "2d5", 200, "fused-e"), (4, "3d7", 36, "fused-e"),
                                                 (3, "3d27", 20, "fused-f"),
                                                 # world = kMaxRanks (solver.cu): the comm-block
                                                 # slot layout and arrival counts at their limit
                                                 (8, "3d7", 48, "fused-e"), (8, "3d7", 40, "fused-a"),
                                                 (8, "3d27", 24, "fused-f"), (8, "3d7", 40, "fused-c"),
                                                 # 125-point: bridged plane windows,
                                                 # 6,859-entry dictionary, 1 CTA/SM
                                                 (2, "p125", 30, "fused-f"), (3, "p125", 30, "fused-e")])
def test_virtual_ranks_match_single_gpu(cuda, world, kind, n, engine):
    A = oracle.stencil(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    out = run_virtual(world, lambda g: D.shard_stencil(kind, n, g), cfg, engine=engine)
    x = np.concatenate([o[0] for o in out])
    reps = [o[1] for o in out]
    assert len({r.iterations for r in reps}) == 1          # ranks agree
    assert all(r.history == reps[0].history for r in reps)  # identical scalars on every rank
    rep = reps[0]
    assert rep.converged
    assert abs(rep.iterations - ref.iterations) <= 1
    assert oracle.history_gap(rep.history, ref.history) <= 1e-10
    assert np.max(np.abs(x - ref.x)) / np.max(np.abs(ref.x)) <= 1e-8
    assert np.max(np.abs(x - x_true)) < 1e-6


def test_virtual_ranks_host_csr_irregular(cuda):
    """shard_csr on a non-stencil SPD matrix (irregular halo sets)."""
    import scipy.sparse as sp

    n = 3000
    M = sp.random(n, n, density=0.003, random_state=11, format="csr")
    M = (M + M.T).tocsr()
    M.data[:] = -np.abs(M.data)
    M = M + sp.diags(np.asarray(np.abs(M).sum(axis=1)).ravel() + 1.0)
    M = M.tocsr()
    M.sort_indices()
    A = pb.CsrMatrix(n, n, M.indptr, M.indices, M.data)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=5000)
    out = run_virtual(3, lambda g: D.shard_csr(A, g), cfg)
    x = np.concatenate([o[0] for o in out])
    rep = out[0][1]
    assert abs(rep.iterations - ref.iterations) <= 1
    assert oracle.history_gap(rep.history, ref.history) <= 1e-10
    assert np.max(np.abs(x - ref.x)) / np.max(np.abs(ref.x)) <= 1e-8


def test_virtual_ranks_repeat_and_max_iterations(cuda):
    """Two solves on the same connected solvers (counters carry over) and an
    iteration cap that ends mid-chunk."""
    kind, n, world = "3d7", 24, 2
    G = D.LocalGroup(world)
    res = [None] * world
    errs = []

    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            prob = D.shard_stencil(kind, n, g)
            solver = D.DistributedSolver(prob, g, pb.DeviceOptions(max_sms=60, chunk=8))
            xt, b = D.manufactured_local(prob)
            reps = []
            for maxit in (5, 13, 2000):
                cfg = pb.SolverConfig(tolerance=1e-10, max_iterations=maxit, record_history=True)
                x, rep = D.pipecg_solve_distributed(prob, b, torch.zeros_like(b), cfg, g,
                                                    solver=solver)
                reps.append((rep, x.cpu().numpy()))
            solver.close()
            res[r] = reps
        except BaseException as e:  # noqa: BLE001
            errs.append((r, repr(e)))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    A = oracle.stencil(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    for k, maxit in enumerate((5, 13, 2000)):
        ref = oracle.pipecg_solve(A, b, x0, d, tol=1e-10, max_iterations=maxit)
        rep = res[0][k][0]
        assert abs(rep.iterations - ref.iterations) <= 1
        assert oracle.history_gap(rep.history, ref.history) <= 1e-10
        x = np.concatenate([res[r][k][1] for r in range(world)])
        assert np.max(np.abs(x - ref.x)) / max(np.max(np.abs(ref.x)), 1e-300) <= 1e-8
        if maxit < 100:
            assert rep.iterations == maxit and not rep.converged


def test_virtual_ranks_e2e_host_blocks_and_autotune_agreement(cuda):
    """The host-buffer multi-GPU call (bench e2e leg at N > 1): each rank
    uploads its own host row block; blocks >= 64K rows autotune per rank and
    must agree on one fused variant (the exchange pushes that variant's
    gathered vector)."""
    kind, n, world = "3d7", 64, 2
    A = oracle.stencil(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    G = D.LocalGroup(world)
    out, errs = [None] * world, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            out[r] = D.e2e_distributed(kind, n, g, tol,
                                       options=pb.DeviceOptions(max_sms=148 // world - 10))
        except BaseException as e:  # noqa: BLE001
            errs.append((r, repr(e)))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    it, secs, h2d, d2h, err = out[0]
    assert abs(it - ref.iterations) <= 1 and secs > 0
    assert err < 1e-6
    assert sum(o[3] for o in out) == 8 * A.n_rows


@pytest.mark.parametrize("engine,code", [("fused-e", 8), ("fused-f", 9)])
def test_virtual_ranks_keep_row_pattern_variants(cuda, engine, code):
    """A stencil shard's dictionary is valid in its [owned | halo] column
    space: E/F stay in use once connected (windows over the halo ranges)."""
    world, n = 2, 40
    G = D.LocalGroup(world)
    opts = pb.DeviceOptions(max_sms=shared_max_sms(world), engine=engine)
    got, errs = [None] * world, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            prob = D.shard_stencil("3d7", n, g)
            s = D.DistributedSolver(prob, g, opts)
            xt, b = D.manufactured_local(prob)
            s.init(b, torch.zeros_like(b), 1e-30, 30)
            res = s.run(False, 30)[0]
            got[r] = (res.engine, res.pattern_flags, res.iterations)
            s.close()
        except BaseException as e:  # noqa: BLE001
            errs.append((r, repr(e)))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    for eng, flags, its in got:
        assert eng == code and flags & 3 == 3 and its == 30


@pytest.mark.parametrize("kind,n", [("3d7", 24), ("2d5", 120)])
def test_pipecg_solve_devices_keyword(cuda, kind, n):
    """pipecg_solve(..., devices=[0, 0]): the one-process multi-device entry
    (the reference's devices= keyword) -- here two ranks sharing the one
    GPU; same iterations and x as the single-device solve, within the
    oracle's reorder envelope."""
    A = pb.stencil_host(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    x, rep = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, devices=[0, 0])
    assert isinstance(x, np.ndarray) and x.shape == (A.n_rows,)
    assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
    assert oracle.history_gap(rep.history, ref.history) <= 1e-10
    assert np.max(np.abs(x - ref.x)) / np.max(np.abs(ref.x)) <= 1e-8
    assert rep.partition["world"] == 2


def test_pipecg_solve_devices_custom_preconditioner(cuda):
    """The caller's inv_diag (not the shard's own Jacobi) is used on every rank."""
    A = pb.stencil_host("3d7", 20)
    x_true, b, x0, d = oracle.manufactured(A)
    d = d.copy()
    d[::7] *= 0.9
    tol = oracle.recipe_tolerance(A, b, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    x, rep = pb.pipecg_solve(A, b, x0, pb.JacobiPreconditioner(d), cfg, devices=[0, 0, 0])
    assert abs(rep.iterations - ref.iterations) <= 1
    assert np.max(np.abs(x - ref.x)) / np.max(np.abs(ref.x)) <= 1e-8


def test_virtual_ranks_config5_shaped(cuda):
    """BASELINE configs[4] in miniature: the 7-pt Poisson matrix sharded 8
    ways with every shard generated on the device from its own row block
    (shard_stencil -> pipecg_b200_stencil_fill; the 1.5B-row case cannot
    exist on the host), solved to the recipe tolerance; iterations, history
    and x against the single-matrix oracle."""
    kind, n, world = "3d7", 56, 8
    A = oracle.stencil(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000)
    out = run_virtual(world, lambda g: D.shard_stencil(kind, n, g), cfg)
    plans = [o[2] for o in out]
    assert sum(p.n_local for p in plans) == n ** 3
    assert all(p.cuts == plans[0].cuts for p in plans) and len(plans[0].cuts) == world + 1
    x = np.concatenate([o[0] for o in out])
    reps = [o[1] for o in out]
    assert len({r.iterations for r in reps}) == 1
    assert all(r.history == reps[0].history for r in reps)
    assert abs(reps[0].iterations - ref.iterations) <= 1
    assert oracle.history_gap(reps[0].history, ref.history) <= 1e-10
    assert np.max(np.abs(x - ref.x)) / np.max(np.abs(ref.x)) <= 1e-8


@pytest.mark.parametrize("world,engine,k", [(2, "fused-e", 3), (3, "fused-a", 1), (2, "fused-f", 2),
                                            (4, "fused-c", 5)])
def test_virtual_ranks_drift_samples(cuda, world, engine, k):
    """Drift samples on a row-sharded solve (solvers.py:190-192,371-372):
    every k iterations each rank pushes its boundary rows of x to the peers
    (double-buffered spare halo), sums ((b - A x) - r)^2 over its rows and
    the ranks' sums are combined in rank order in-kernel.  Same sample
    iterations as the oracle, identical values on every rank, the reference
    test's bound, and close to the oracle's own samples."""
    kind, n = "3d7", 24
    A = oracle.stencil(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True,
                          drift_check_interval=k)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000, drift_check_interval=k)
    out = run_virtual(world, lambda g: D.shard_stencil(kind, n, g), cfg, engine=engine)
    reps = [o[1] for o in out]
    dh = reps[0].drift_history
    assert dh and all(r.drift_history == dh for r in reps)
    assert [it for it, _ in dh] == [it for it, _ in ref.drift_history][: len(dh)]
    assert abs(len(dh) - len(ref.drift_history)) <= 1
    bn = float(np.linalg.norm(b))
    for (it, v), (_, vr) in zip(dh, ref.drift_history):
        assert v <= 1e-10 * max(1.0, bn)
        assert abs(v - vr) <= 1e-12 * max(1.0, bn), (it, v, vr)


def test_destroy_while_peer_waits_does_not_stall(cuda):
    """A rank's thread destroys an unrelated solver while its peer's kernel
    already waits for this rank's first arrival (virtual ranks, one GPU).
    cudaFree synchronises the whole device, so an immediate free would block
    this thread until the peer's spin timed out (10 s, 'exchange timed
    out'); the library parks such frees while connected solvers live."""
    import time

    kind, n, world = "3d7", 24, 2
    G = D.LocalGroup(world)
    other = pb.PipecgSolver(pb.stencil_device("3d7", 16),
                            pb.jacobi_setup(pb.stencil_device("3d7", 16)).inv_diag,
                            pb.DeviceOptions(max_sms=20))
    started = threading.Event()
    res, errs, waited = [None] * world, [], []

    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            prob = D.shard_stencil(kind, n, g)
            solver = D.DistributedSolver(prob, g, pb.DeviceOptions(max_sms=shared_max_sms(world)))
            xt, b = D.manufactured_local(prob)
            solver.init(b, torch.zeros_like(b), 1e-10, 2000)
            torch.cuda.ExternalStream(solver.stream).synchronize()
            if r == 0:
                started.set()
            else:
                started.wait(30)
                time.sleep(0.3)  # rank 0's iteration-1 kernel now spins on our arrival
                t = time.perf_counter()
                other.close()
                waited.append(time.perf_counter() - t)
            out = solver.run(False, 2000)
            res[r] = out[0]
            solver.close()
        except BaseException as e:  # noqa: BLE001
            errs.append((r, repr(e)))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not errs, errs
    assert waited and waited[0] < 2.0, waited
    assert res[0].converged and res[0].iterations == res[1].iterations


def test_connected_e_runs_the_staged_layout(cuda):
    """A connected E never keeps the consumer-loaded stage layout (pattern
    flag 32) the single-GPU autotuner may pick: with the fused exchange it
    measured 1.5-1.6x slower (tools/dist1.py; csrc/solver.cu
    solver_connect).  And an autotuned engine runs as E, not F, once
    connected (distributed.py)."""
    for engine in ("fused-e", "fused"):
        G = D.LocalGroup(1)
        g = G.view(0)
        prob = D.shard_stencil("3d7", 128, g)
        s = D.DistributedSolver(prob, g, pb.DeviceOptions(engine=engine))
        xt, b = D.manufactured_local(prob)
        s.init(b, torch.zeros_like(b), 1e-9, 50)
        res = s.run(False, 50)[0]
        assert res.engine == 8, (engine, res.engine)
        assert not (res.pattern_flags & 32), (engine, res.pattern_flags)
        s.close()
