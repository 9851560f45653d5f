"""ctypes front end of the CPU oracle (oracle/pipecg_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker for tests/, the check inside
``__graft_entry__.smoke()`` and the CPU baseline leg of ``bench.py``.  The
product package ``paper_2105_06176_b200`` must never import this module.

Each function restates one reference function (file:line relative to
/root/reference/pkg/src/pipecg) and is pinned to the reference's own outputs
by ``tests/golden`` (see ``tests/test_oracle.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libpipecg_oracle.so"
_lib = None

OR_OK = 0
BREAKDOWN_NAMES = {1: "alpha denominator", 2: "gamma", 3: "delta"}

_p_i64 = ctypes.POINTER(ctypes.c_int64)
_p_f64 = ctypes.POINTER(ctypes.c_double)


class _Report(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("final_norm", ctypes.c_double),
        ("converged", ctypes.c_int),
        ("status", ctypes.c_int),
        ("bd_iteration", ctypes.c_int64),
        ("bd_value", ctypes.c_double),
        ("n_drift", ctypes.c_int64),
    ]


def build() -> Path:
    """Compile the oracle with its Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.or_spmv.argtypes = [ctypes.c_int64, _p_i64, _p_i64, _p_f64, _p_f64, _p_f64]
        L.or_dot_seq.argtypes = [ctypes.c_int64, _p_f64, _p_f64]
        L.or_dot_seq.restype = ctypes.c_double
        L.or_dot_blocked.argtypes = [ctypes.c_int64, _p_f64, _p_f64]
        L.or_dot_blocked.restype = ctypes.c_double
        L.or_fused_update.argtypes = [ctypes.c_int64] + [_p_f64] * 10 + [ctypes.c_double] * 2
        L.or_jacobi_apply.argtypes = [ctypes.c_int64, _p_f64, _p_f64, _p_f64]
        L.or_pipecg_scalars.argtypes = [ctypes.c_double] * 4 + [ctypes.c_int64] + [_p_f64] * 3
        L.or_pipecg_scalars.restype = ctypes.c_int
        L.or_pipecg_solve.argtypes = (
            [ctypes.c_int64, _p_i64, _p_i64, _p_f64, _p_f64, _p_f64, _p_f64,
             ctypes.c_double, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
             _p_f64, _p_f64, _p_i64, _p_f64, _p_f64, ctypes.POINTER(_Report)]
        )
        L.or_pipecg_solve.restype = ctypes.c_int
        L.or_pcg_solve.argtypes = (
            [ctypes.c_int64, _p_i64, _p_i64, _p_f64, _p_f64, _p_f64, _p_f64,
             ctypes.c_double, ctypes.c_int64, ctypes.c_int, _p_f64, _p_f64,
             ctypes.POINTER(_Report)]
        )
        L.or_pcg_solve.restype = ctypes.c_int
        L.or_set_threads.argtypes = [ctypes.c_int]
        L.or_set_exact_dots.argtypes = [ctypes.c_int]
        L.or_max_threads.restype = ctypes.c_int
        L.or_gen_csr.argtypes = [ctypes.c_int, ctypes.c_int64, _p_i64, _p_i64, _p_f64]
        L.or_gen_csr.restype = ctypes.c_int
        L.or_stepper_begin.argtypes = [ctypes.c_int64, _p_i64, _p_i64, _p_f64, _p_f64, _p_f64]
        L.or_stepper_begin.restype = ctypes.c_void_p
        L.or_stepper_steps.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.or_stepper_steps.restype = ctypes.c_int
        L.or_stepper_norm.argtypes = [ctypes.c_void_p]
        L.or_stepper_norm.restype = ctypes.c_double
        L.or_stepper_end.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=_p_f64):
    return None if a is None else a.ctypes.data_as(t)


def set_threads(t: int) -> int:
    """Thread count for the CPU baseline (1 = the reference's own orders)."""
    lib().or_set_threads(int(t))
    return int(t)


def set_exact_dots(exact: bool) -> None:
    """True (default): dots in the requested order (seq = the reference's)
    for any thread count.  False: static-chunked parallel dots -- only for
    the CPU-baseline timing (bench.py), never for parity."""
    lib().or_set_exact_dots(1 if exact else 0)


def max_threads() -> int:
    return int(lib().or_max_threads())


@dataclass
class Csr:
    """Plain host CSR with the reference's dtypes (sparse.py:59-71)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])


def as_csr(A) -> Csr:
    """Accept any CsrMatrix-like object (duck-typed, sparse.py:43-71)."""
    return Csr(
        int(A.n_rows), int(A.n_cols),
        np.ascontiguousarray(A.row_offsets, dtype=np.int64),
        np.ascontiguousarray(A.col_indices, dtype=np.int64),
        np.ascontiguousarray(A.values, dtype=np.float64),
    )


# --- kernels.py ------------------------------------------------------------

def spmv(A, x) -> np.ndarray:
    """kernels.py:64-70 / 152-164."""
    A = as_csr(A)
    x = _f64(x)
    out = np.empty(A.n_rows)
    lib().or_spmv(A.n_rows, _ptr(A.row_offsets, _p_i64), _ptr(A.col_indices, _p_i64),
                  _ptr(A.values), _ptr(x), _ptr(out))
    return out


def dot(a, b) -> float:
    """kernels.py:92-97 / 192-196 (strict left-to-right)."""
    a, b = _f64(a), _f64(b)
    assert a.shape == b.shape
    return float(lib().or_dot_seq(a.size, _ptr(a), _ptr(b)))


def dot_blocked(a, b) -> float:
    """Reorder-only dot (256 sequential partials + tree); noise-floor probe."""
    a, b = _f64(a), _f64(b)
    return float(lib().or_dot_blocked(a.size, _ptr(a), _ptr(b)))


def norm2(a) -> float:
    """kernels.py:199-201."""
    return float(np.sqrt(dot(a, a)))


def fused_update(v: dict, alpha: float, beta: float) -> dict:
    """kernels.py:100-111 on copies of the ten state vectors in ``v``."""
    out = {k: _f64(v[k]).copy() for k in ("z", "q", "s", "p", "x", "r", "u", "w", "m", "n")}
    n = out["x"].size
    lib().or_fused_update(
        n, *[_ptr(out[k]) for k in ("z", "q", "s", "p", "x", "r", "u", "w", "m", "n")],
        float(alpha), float(beta),
    )
    return out


def jacobi_apply(inv_diag, v) -> np.ndarray:
    """kernels.py:240-247."""
    d, v = _f64(inv_diag), _f64(v)
    out = np.empty_like(v)
    lib().or_jacobi_apply(v.size, _ptr(d), _ptr(v), _ptr(out))
    return out


def jacobi_inv_diag(A) -> np.ndarray:
    """kernels.py:218-237 (diagonal extraction + reciprocal, no error paths)."""
    A = as_csr(A)
    rows = np.repeat(np.arange(A.n_rows, dtype=np.int64), np.diff(A.row_offsets))
    on = A.col_indices == rows
    diag = np.zeros(A.n_rows)
    diag[rows[on]] = A.values[on]
    return 1.0 / diag


# --- solvers.py ------------------------------------------------------------

def pipecg_scalars(gamma, gamma_prev, delta, alpha_prev, iteration):
    """solvers.py:276-294.  Returns (alpha, beta) or ("breakdown", denom)."""
    a, b, bad = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    rc = lib().or_pipecg_scalars(float(gamma), float(gamma_prev), float(delta),
                                 float(alpha_prev), int(iteration),
                                 ctypes.byref(a), ctypes.byref(b), ctypes.byref(bad))
    if rc != OR_OK:
        return ("breakdown", bad.value)
    return a.value, b.value


@dataclass
class OracleResult:
    x: np.ndarray
    iterations: int
    final_norm: float
    converged: bool
    history: list | None
    drift_history: list | None
    breakdown: tuple | None = None  # (quantity, iteration, value)
    state: dict | None = field(default=None, repr=False)


def pipecg_solve(A, b, x0, inv_diag, tol=1e-5, max_iterations=10000,
                 record_history=True, drift_check_interval=0, dot_mode="seq",
                 want_state=False) -> OracleResult:
    """solvers.py:297-387 (pipecg_init + pipecg_solve)."""
    A = as_csr(A)
    N = A.n_rows
    b, x0, d = _f64(b), _f64(x0), _f64(inv_diag)
    x = np.empty(N)
    hist = np.empty(max_iterations + 1) if record_history else None
    nd = max_iterations // drift_check_interval + 1 if drift_check_interval > 0 else 0
    d_it = np.zeros(nd, dtype=np.int64) if nd else None
    d_val = np.zeros(nd) if nd else None
    state = np.empty(10 * N) if want_state else None
    rep = _Report()
    lib().or_pipecg_solve(
        N, _ptr(A.row_offsets, _p_i64), _ptr(A.col_indices, _p_i64), _ptr(A.values),
        _ptr(b), _ptr(x0), _ptr(d), float(tol), int(max_iterations),
        int(drift_check_interval), 1 if dot_mode == "blocked" else 0,
        _ptr(x), _ptr(hist), _ptr(d_it, _p_i64), _ptr(d_val), _ptr(state),
        ctypes.byref(rep),
    )
    bd = None
    if rep.status != OR_OK:
        bd = (BREAKDOWN_NAMES.get(rep.status, "error"), int(rep.bd_iteration), float(rep.bd_value))
    history = None
    if record_history and bd is None:
        history = hist[: rep.iterations + 1].tolist()
    drift = None
    if drift_check_interval > 0:
        drift = [[int(d_it[k]), float(d_val[k])] for k in range(rep.n_drift)]
    st = None
    if want_state:
        names = ("x", "r", "u", "w", "m", "n", "z", "q", "s", "p")
        st = {k: state[i * N:(i + 1) * N].copy() for i, k in enumerate(names)}
    return OracleResult(x, int(rep.iterations), float(rep.final_norm), bool(rep.converged),
                        history, drift, bd, st)


def pcg_solve(A, b, x0, inv_diag, tol=1e-5, max_iterations=10000,
              dot_mode="seq") -> OracleResult:
    """solvers.py:195-273."""
    A = as_csr(A)
    N = A.n_rows
    b, x0, d = _f64(b), _f64(x0), _f64(inv_diag)
    x = np.empty(N)
    hist = np.empty(max_iterations + 1)
    rep = _Report()
    lib().or_pcg_solve(
        N, _ptr(A.row_offsets, _p_i64), _ptr(A.col_indices, _p_i64), _ptr(A.values),
        _ptr(b), _ptr(x0), _ptr(d), float(tol), int(max_iterations),
        1 if dot_mode == "blocked" else 0, _ptr(x), _ptr(hist), ctypes.byref(rep),
    )
    bd = None
    if rep.status != OR_OK:
        bd = (BREAKDOWN_NAMES.get(rep.status, "error"), int(rep.bd_iteration), float(rep.bd_value))
    return OracleResult(x, int(rep.iterations), float(rep.final_norm), bool(rep.converged),
                        hist[: rep.iterations + 1].tolist() if bd is None else None, None, bd)


# --- problem recipes (cli.py:83-100) ------------------------

STENCILS = {"2d5": 5, "3d7": 7, "3d27": 27, "p125": 125}


def stencil(kind: str, n: int) -> Csr:
    """x-fastest natural-order stencil matrix, ascending columns."""
    k = STENCILS[kind]
    N = n * n if k == 5 else n ** 3
    ro = np.empty(N + 1, dtype=np.int64)
    lib().or_gen_csr(k, n, _ptr(ro, _p_i64), None, None)
    nnz = int(ro[-1])
    ci = np.empty(nnz, dtype=np.int64)
    va = np.empty(nnz)
    lib().or_gen_csr(k, n, _ptr(ro, _p_i64), _ptr(ci, _p_i64), _ptr(va))
    return Csr(N, N, ro, ci, va)


def row_patterns(A, max_pat=256, max_entries=8192):
    """Checker for the device row-pattern dictionary (csrc/patterns.cu): the
    distinct rows of A written relative to their own index -- (col - i,
    value bits) in CSR order -- numbered by first occurrence.  Returns
    (n_pat, n_entries, codes uint8[n]) or (0, 0, None) when there are more
    than max_pat lists or max_entries entries.  Not a reference function:
    the dictionary is a storage format of the reference's CSR
    (sparse.py:43-132), whose SpMV order (kernels.py:64-70) it preserves."""
    A = as_csr(A)
    ro, ci, va = A.row_offsets, A.col_indices, np.ascontiguousarray(A.values).view(np.int64)
    seen, codes, entries = {}, np.empty(A.n_rows, dtype=np.uint8), 0
    for i in range(A.n_rows):
        lo, hi = int(ro[i]), int(ro[i + 1])
        key = (tuple((ci[lo:hi] - i).tolist()), tuple(va[lo:hi].tolist()))
        c = seen.get(key)
        if c is None:
            if len(seen) == max_pat:
                return 0, 0, None
            c = seen[key] = len(seen)
            entries += hi - lo
        codes[i] = c
    if entries > max_entries:
        return 0, 0, None
    return len(seen), entries, codes


def manufactured(A):
    """cli.py:83-100: x_true = 1/sqrt(N), b = A x_true, x0 = 0, Jacobi."""
    N = A.n_rows
    x_true = np.full(N, 1.0 / np.sqrt(N))
    b = spmv(A, x_true)
    return x_true, b, np.zeros(N), jacobi_inv_diag(A)


def recipe_tolerance(A, b, inv_diag) -> float:
    """tolerance = 1e-8 * sqrt((u0,u0)) with u0 = M^{-1}(b - A*0)."""
    u0 = jacobi_apply(inv_diag, b)
    return 1e-8 * math.sqrt(dot(u0, u0))


def history_gap(h_test, h_ref) -> float:
    """G = max_k |h_k - h_k^ref| / h_0 over the common prefix."""
    k = min(len(h_test), len(h_ref))
    a = np.asarray(h_test[:k])
    r = np.asarray(h_ref[:k])
    return float(np.max(np.abs(a - r)) / h_ref[0]) if k else 0.0


class Stepper:
    """pipecg_init once, then fixed-count iterations (CPU baseline timing only)."""

    def __init__(self, A, b, inv_diag):
        self.A = as_csr(A)
        self.b = _f64(b)
        self.d = _f64(inv_diag)
        self.h = lib().or_stepper_begin(
            self.A.n_rows, _ptr(self.A.row_offsets, _p_i64), _ptr(self.A.col_indices, _p_i64),
            _ptr(self.A.values), _ptr(self.b), _ptr(self.d))
        if not self.h:
            raise MemoryError("oracle stepper allocation failed")

    def steps(self, count: int) -> None:
        rc = lib().or_stepper_steps(self.h, int(count))
        if rc:
            raise RuntimeError(f"oracle breakdown {BREAKDOWN_NAMES.get(rc, rc)}")

    def norm(self) -> float:
        return float(lib().or_stepper_norm(self.h))

    def close(self):
        if self.h:
            lib().or_stepper_end(self.h)
            self.h = None

    def __del__(self):
        self.close()


def lib_path() -> str:
    return os.fspath(_LIB_PATH)


# --- sparse.py:183-326 (Matrix Market) -------------------------------------

class MMError(ValueError):
    """Oracle form of MatrixMarketError (sparse.py:29-36): message + line."""

    def __init__(self, message, line):
        self.line_number = line
        super().__init__(f"line {line}: {message}")


def _mm_float(tok, line):
    # sparse.py:183-192: Python float(), then the Fortran 'd' exponent retry
    try:
        return float(tok)
    except ValueError:
        try:
            return float(tok.replace("d", "e").replace("D", "E"))
        except ValueError:
            raise MMError(f"bad value {tok!r}", line) from None


def _np_pairwise(a):
    """numpy's pairwise_sum for float64 (what np.add.reduceat applies to a
    segment after its first element): < 8 terms sequential from 0.0,
    <= 128 eight interleaved accumulators, else halves (multiple of 8)."""
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r = r + x
        return r
    if n <= 128:
        r = list(a[:8])
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] = r[j] + a[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for x in a[i:]:
            res = res + x
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _np_pairwise(a[:n2]) + _np_pairwise(a[n2:])


def parse_matrix_market(text: str) -> Csr:
    """Restatement of parse_matrix_market (sparse.py:195-320): header and
    size checks in the reference's order, 1-based line numbers, symmetric
    mirroring, (row, col) stable sort, duplicates summed like the
    reference's np.add.reduceat (numpy 2.x pairwise order)."""
    if not text:
        raise MMError("empty document", 1)
    lines = text.split("\n")
    if text.endswith("\n"):
        lines = lines[:-1]
    tok = lines[0].strip().lower().split()
    if len(tok) < 5 or tok[0] != "%%matrixmarket":
        raise MMError("missing %%MatrixMarket header", 1)
    checks = (("matrix", "object"), ("coordinate", "format"), ("real", "field"))
    for k, (want, what) in enumerate(checks, start=1):
        if tok[k] != want:
            raise MMError(f"unsupported {what} {tok[k]!r}", 1)
    if tok[4] not in ("general", "symmetric"):
        raise MMError(f"unsupported symmetry {tok[4]!r}", 1)
    sym = tok[4] == "symmetric"
    k = 1
    while k < len(lines) and (not lines[k].strip() or lines[k].strip().startswith("%")):
        k += 1
    if k >= len(lines):
        raise MMError("missing size line", 2)
    size_no = k + 1
    parts = lines[k].split()
    if len(parts) != 3:
        raise MMError("size line must hold rows cols entries", size_no)
    try:
        nr, nc, ne = (int(p) for p in parts)
    except ValueError:
        raise MMError("size line must hold three integers", size_no) from None
    if nr <= 0 or nc <= 0 or ne <= 0:
        raise MMError("empty matrix", size_no)
    if sym and nr != nc:
        raise MMError("symmetric matrix must be square", size_no)
    rows, cols, vals = [], [], []
    last = size_no
    for ln in range(k + 1, len(lines)):
        t = lines[ln].strip()
        if not t or t.startswith("%"):
            continue
        no = ln + 1
        if len(rows) >= ne:
            raise MMError(f"more than the declared {ne} entries", no)
        p = t.split()
        if len(p) != 3:
            raise MMError("entry must hold row col value", no)
        try:
            i, j = int(p[0]), int(p[1])
        except ValueError:
            raise MMError("bad coordinate", no) from None
        if not 1 <= i <= nr:
            raise MMError(f"row index {i} out of range", no)
        if not 1 <= j <= nc:
            raise MMError(f"column index {j} out of range", no)
        vals.append(_mm_float(p[2], no))
        rows.append(i - 1)
        cols.append(j - 1)
        last = no
    if len(rows) != ne:
        raise MMError(f"expected {ne} entries, found {len(rows)}", last + 1)
    r = np.array(rows, dtype=np.int64)
    c = np.array(cols, dtype=np.int64)
    v = np.array(vals, dtype=np.float64)
    if sym:
        off = r != c
        r, c, v = np.concatenate([r, c[off]]), np.concatenate([c, r[off]]), np.concatenate([v, v[off]])
    key = r * nc + c
    order = np.argsort(key, kind="stable")
    key, v = key[order], v[order]
    heads = np.flatnonzero(np.r_[True, key[1:] != key[:-1]])
    bounds = np.r_[heads, key.size]
    sums = np.empty(heads.size)
    for s in range(heads.size):  # np.add.reduceat order: first + pairwise(rest)
        seg = [float(x) for x in v[bounds[s]:bounds[s + 1]]]
        sums[s] = seg[0] + _np_pairwise(seg[1:])
    ro = np.zeros(nr + 1, dtype=np.int64)
    np.cumsum(np.bincount(key[heads] // nc, minlength=nr), out=ro[1:])
    return Csr(nr, nc, ro, key[heads] % nc, sums)
