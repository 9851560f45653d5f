"""Config-scale goldens: tests/golden/config_scale/<name>.npz (+ .json).

Run in the dev container (the reference exists only here):

    python tests/golden/make_config_goldens.py [name ...]

For each BASELINE / north-star configuration at full size this records what
the GPU parity tests (tests/test_gpu_config_scale.py, ``-m "gpu and slow"``)
compare against:

* the reference-order history (``history``: iterations + 1 norms) and the
  iteration count of the recipe solve (x_true = 1/sqrt(N), b = A x_true,
  x0 = 0, Jacobi, tol = 1e-8 * sqrt((u0, u0)));
* the reorder envelope E = max_k |h_k^blocked - h_k| / h_0, where
  ``h^blocked`` is the SAME algorithm with only the dot products reordered
  (256 sequential partials + a tree: oracle ``dot_mode="blocked"``) --
  BASELINE.md gate 2 allows G <= max(1e-10, 3E) for a parallel reduction;
* x: sha256 of the reference-order x (the seq-mode GPU run must match it
  bit for bit), a strided sample of 65,536 entries, and the x gap of the
  reordered run (the envelope for gate 3).

The oracle (oracle/pipecg_oracle.c, checker only) computes them.  Where the
reference itself finishes in minutes here (3D 7-pt 128^3 and 256^3) the
reference is run too and the oracle's history and x must equal it bit for
bit -- the oracle is then pinned at config scale, not only on the small
fixtures of make_golden.py.  The 400^3 configurations are too large for the
reference (hours); there the oracle's own multi-threaded run is the golden.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "config_scale"
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402  (checker)

N_SAMPLE = 65536

# name -> (kind, n, pin with the reference?)
CONFIGS = {
    "3d7-128": ("3d7", 128, True),
    "3d27-64": ("3d27", 64, False),
    "3d27-100": ("3d27", 100, False),
    "powerlaw-22": ("powerlaw", 22, False),
    "3d7-256": ("3d7", 256, True),
    "3d7-400": ("3d7", 400, False),
    "3d27-400": ("3d27", 400, False),
    # the paper's own 125-point Poisson matrices (Table II: n = 165-185)
    "p125-64": ("p125", 64, True),
    "p125-185": ("p125", 185, False),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_idx(N: int) -> np.ndarray:
    k = min(N, N_SAMPLE)
    return np.unique(np.linspace(0, N - 1, k).astype(np.int64))


def problem(kind: str, n: int):
    if kind == "powerlaw":
        from paper_2105_06176_b200.sparse import generate_powerlaw  # host numpy recipe

        A = generate_powerlaw(2 ** n)
        return oracle.as_csr(A)
    return oracle.stencil(kind, n)


def reference_solve(A, b, inv_diag, tol):
    """The reference's own pipecg_solve (solvers.py:324-387) on the same CSR."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
    sys.path.insert(0, "/root/reference/pkg/src")
    import pipecg

    Ar = pipecg.CsrMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, A.values)
    pc = pipecg.JacobiPreconditioner(inv_diag) if hasattr(pipecg, "JacobiPreconditioner") \
        else pipecg.jacobi_setup(Ar)
    cfg = pipecg.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    x, rep = pipecg.pipecg_solve(Ar, b, np.zeros(A.n_rows), pc, cfg)
    return x, rep


def make(name: str) -> dict:
    kind, n, pin = CONFIGS[name]
    t0 = time.time()
    oracle.set_threads(os.cpu_count() or 1)
    A = problem(kind, n)
    N, nnz = A.n_rows, A.nnz
    x_true, b, x0, d = oracle.manufactured(A)
    tol = oracle.recipe_tolerance(A, b, d)
    seq = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000, dot_mode="seq")
    blk = oracle.pipecg_solve(A, b, x0, d, tol=tol, max_iterations=20000, dot_mode="blocked")
    h = np.asarray(seq.history)
    hb = np.asarray(blk.history)
    k = min(h.size, hb.size)
    E = float(np.max(np.abs(hb[:k] - h[:k])) / h[0])
    xs = float(np.max(np.abs(seq.x)))
    x_gap = float(np.max(np.abs(blk.x - seq.x)) / xs)
    idx = sample_idx(N)
    meta = {
        "name": name, "kind": kind, "n": n, "N": int(N), "nnz": int(nnz),
        "tol": tol, "norm0": float(h[0]), "iterations": seq.iterations,
        "iterations_blocked": blk.iterations, "converged": bool(seq.converged),
        "final_norm": seq.final_norm, "E": E, "x_gap_blocked": x_gap,
        "x_sha256": sha(seq.x), "x_inf_err_vs_true": float(np.max(np.abs(seq.x - x_true))),
        "matrix_sha256": sha(A.row_offsets) + ":" + sha(A.col_indices) + ":" + sha(A.values),
        "oracle_threads": os.cpu_count(), "pinned_by_reference": False,
    }
    if pin:
        xr, rep = reference_solve(A, b, d, tol)
        same_h = rep.history == seq.history
        same_x = bool(np.array_equal(xr, seq.x))
        meta["pinned_by_reference"] = bool(same_h and same_x)
        meta["reference_iterations"] = rep.iterations
        meta["reference_phase_times"] = rep.phase_times
        assert same_h and same_x, f"{name}: oracle differs from the reference at config scale"
    np.savez_compressed(OUT / f"{name}.npz", history=h, history_blocked=hb, x_idx=idx,
                        x_sample=seq.x[idx], x_blocked_sample=blk.x[idx])
    meta["seconds"] = time.time() - t0
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1, sort_keys=True))
    print(json.dumps(meta), flush=True)
    return meta


def main(argv):
    OUT.mkdir(exist_ok=True)
    oracle.build()
    names = argv or list(CONFIGS)
    for nm in names:
        make(nm)


if __name__ == "__main__":
    main(sys.argv[1:])
