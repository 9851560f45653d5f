"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run in the dev container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/pipecg (numba needs a writable
NUMBA_CACHE_DIR), runs the reference kernels and solvers on small seeded
inputs, and writes the inputs + outputs as fixtures.  The GPU box never
reads /root/reference; it only reads these fixtures.  The oracle
(oracle/pipecg_oracle.c) and the CUDA path are both checked against them.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, str(REF_SRC))

import pipecg  # noqa: E402  (the reference)
from pipecg import (  # noqa: E402
    SolverBreakdown, SolverConfig, csr_from_dense, dot, fused_pipecg_update,
    generate_poisson125, jacobi_apply, jacobi_setup, pcg_solve, pipecg_solve, spmv,
)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def kron_stencil(kind: str, n: int):
    import scipy.sparse as sp

    if kind == "2d5":
        T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n))
        I = sp.identity(n)
        A = (sp.kron(I, T) + sp.kron(T, I)).tocsr()
    elif kind == "3d7":
        T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(n, n))
        I = sp.identity(n)
        A = (sp.kron(sp.kron(I, I), T) + sp.kron(sp.kron(I, T), I) + sp.kron(sp.kron(T, I), I)).tocsr()
    elif kind == "3d27":
        B = sp.diags([1.0, 1.0, 1.0], [-1, 0, 1], shape=(n, n))
        A = (27.0 * sp.identity(n ** 3) - sp.kron(sp.kron(B, B), B)).tocsr()
    else:
        raise ValueError(kind)
    A.sort_indices()
    A.eliminate_zeros()
    return pipecg.CsrMatrix(A.shape[0], A.shape[1], A.indptr, A.indices, A.data)


def manufactured(A):
    n = A.n_rows
    x_true = np.full(n, 1.0 / np.sqrt(n))
    b = spmv(A, x_true)
    return x_true, b, np.zeros(n), jacobi_setup(A)


def recipe_tol(A, b, pc):
    u0 = jacobi_apply(pc, b - spmv(A, np.zeros(A.n_rows)))
    return 1e-8 * math.sqrt(dot(u0, u0))


def random_spd_dense(rng, n, cond):
    # tests/conftest.py:92-104 of the reference
    lam = np.exp(rng.uniform(0.0, np.log(cond), n))
    spread = lam.max() - lam.min()
    lam = 1.0 + (lam - lam.min()) / (spread + 1e-300) * (cond - 1.0)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    dense = (q * lam) @ q.T
    return (dense + dense.T) / 2.0


def save_matrix(prefix, A, out):
    out[prefix + "_ro"] = np.asarray(A.row_offsets, dtype=np.int64)
    out[prefix + "_ci"] = np.asarray(A.col_indices, dtype=np.int64)
    out[prefix + "_va"] = np.asarray(A.values, dtype=np.float64)


def main():
    meta = {"reference": str(REF_SRC / "pipecg"), "numba": __import__("numba").__version__,
            "numpy": np.__version__, "cases": {}}

    # 1. kernels: fused update, dot, spmv, jacobi ------------------------------
    rng = np.random.default_rng(20261017)
    k = {}
    n = 4099
    names = ("z", "q", "s", "p", "x", "r", "u", "w", "m", "n")
    for nm in names:
        k["in_" + nm] = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)
    alpha, beta = 0.7364301, -1.21875013
    st = type("S", (), {})()
    for nm in names:
        setattr(st, nm, k["in_" + nm].copy())
    fused_pipecg_update(st, alpha, beta)
    for nm in names:
        k["out_" + nm] = getattr(st, nm)
    k["alpha"] = np.array(alpha)
    k["beta"] = np.array(beta)
    a = rng.standard_normal(2000) * 10.0 ** rng.integers(-8, 8, 2000)
    b = rng.standard_normal(2000) * 10.0 ** rng.integers(-8, 8, 2000)
    k["dot_a"], k["dot_b"] = a, b
    k["dot_ab"] = np.array(dot(a, b))
    P6 = generate_poisson125(6)
    save_matrix("p125n6", P6, k)
    xs = np.random.default_rng(12).standard_normal(P6.n_cols)
    k["p125n6_x"] = xs
    k["p125n6_y"] = spmv(P6, xs)
    pc6 = jacobi_setup(P6)
    k["p125n6_inv_diag"] = pc6.inv_diag
    k["p125n6_jacobi"] = jacobi_apply(pc6, xs)
    # random sparse non-symmetric CSR (test_kernels.py:66-76 style)
    dense = np.where(rng.random((37, 29)) < 0.3, rng.standard_normal((37, 29)), 0.0)
    R = csr_from_dense(dense)
    save_matrix("rand", R, k)
    k["rand_shape"] = np.array([37, 29])
    xr = rng.standard_normal(29)
    k["rand_x"] = xr
    k["rand_y"] = spmv(R, xr)
    np.savez_compressed(HERE / "kernels.npz", **k)

    # 2. stencil structure: reference-style (kron) matrices -> sha256 ----------
    st_meta = {}
    for kind, nn in (("2d5", 33), ("3d7", 11), ("3d27", 9)):
        A = kron_stencil(kind, nn)
        st_meta[f"{kind}_{nn}"] = {"N": A.n_rows, "nnz": A.nnz,
                                   "sha256": sha(A.row_offsets, A.col_indices, A.values)}
    P7 = generate_poisson125(7)
    st_meta["p125_7"] = {"N": P7.n_rows, "nnz": P7.nnz,
                         "sha256": sha(P7.row_offsets, P7.col_indices, P7.values)}
    meta["stencils"] = st_meta

    # 3. solves ------------------------------------------------------------------
    solves = {}

    def record(name, A, b, x0, pc, cfg, solver=pipecg_solve, keep_matrix=True):
        out = {}
        if keep_matrix:
            save_matrix("A", A, out)
        out["b"], out["x0"], out["inv_diag"] = b, x0, pc.inv_diag
        out["tol"] = np.array(cfg.tolerance)
        out["max_iterations"] = np.array(cfg.max_iterations)
        out["drift_k"] = np.array(cfg.drift_check_interval)
        try:
            x, rep = solver(A, b, x0, pc, cfg)
        except SolverBreakdown as e:
            out["breakdown"] = np.array([e.iteration, e.value])
            solves[name] = {"breakdown": e.quantity, "iteration": e.iteration, "value": e.value}
            np.savez_compressed(HERE / f"solve_{name}.npz", **out)
            return
        out["x"] = x
        out["history"] = np.array(rep.history if rep.history is not None else [])
        out["drift"] = np.array(rep.drift_history if rep.drift_history else np.zeros((0, 2)))
        solves[name] = {"iterations": rep.iterations, "converged": rep.converged,
                        "final_norm": rep.final_norm, "strategy": rep.strategy}
        np.savez_compressed(HERE / f"solve_{name}.npz", **out)

    P6 = generate_poisson125(6)
    _, b6, x06, pc6 = manufactured(P6)
    record("p125n6_default", P6, b6, x06, pc6, SolverConfig(record_history=True))
    record("p125n6_drift", P6, b6, x06, pc6,
           SolverConfig(tolerance=1e-9, record_history=True, drift_check_interval=2))
    record("p125n6_pcg", P6, b6, x06, pc6, SolverConfig(record_history=True), solver=pcg_solve)
    for kind, nn in (("2d5", 64), ("3d7", 16)):
        A = kron_stencil(kind, nn)
        _, bb, x0, pc = manufactured(A)
        record(f"{kind}_{nn}", A, bb, x0, pc,
               SolverConfig(tolerance=recipe_tol(A, bb, pc), max_iterations=20000,
                            record_history=True))
    rng = np.random.default_rng(42)
    D = random_spd_dense(rng, 30, 15.0)
    A = csr_from_dense(D)
    xt = rng.standard_normal(30)
    bD = D @ xt
    record("spd30", A, bD, np.zeros(30), jacobi_setup(A),
           SolverConfig(tolerance=1e-8, max_iterations=200, record_history=True))
    A2 = csr_from_dense(np.array([[4.0, 1.0], [1.0, 3.0]]))
    record("spd2", A2, np.array([1.0, 2.0]), np.zeros(2), jacobi_setup(A2),
           SolverConfig(record_history=True))
    Ai = csr_from_dense(np.diag([1.0, -1.0]))
    record("indefinite", Ai, np.ones(2), np.zeros(2), jacobi_setup(Ai), SolverConfig())
    # nonzero x0 + max_iterations cut (not converged)
    rngx = np.random.default_rng(7)
    record("p125n6_cut", P6, b6, rngx.standard_normal(P6.n_rows), pc6,
           SolverConfig(max_iterations=5, record_history=True))
    meta["cases"] = solves

    # 4. config 1 (2D 5-pt 512^2), the reference's CPU-runnable headline config --
    A = kron_stencil("2d5", 512)
    _, bb, x0, pc = manufactured(A)
    tol = recipe_tol(A, bb, pc)
    x, rep = pipecg_solve(A, bb, x0, pc, SolverConfig(tolerance=tol, max_iterations=20000,
                                                      record_history=True))
    np.savez_compressed(HERE / "config1_2d5_512.npz", history=np.array(rep.history),
                        x=x, tol=np.array(tol))
    meta["config1"] = {"iterations": rep.iterations, "final_norm": rep.final_norm,
                       "tol": tol, "norm0": rep.history[0],
                       "phase_times": rep.phase_times}
    (HERE / "golden_meta.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(json.dumps({k: v for k, v in meta.items() if k != "stencils"}, indent=1))


if __name__ == "__main__":
    main()
