"""CSR storage: the reference's host ``CsrMatrix`` plus its device form.

``CsrMatrix`` mirrors /root/reference/pkg/src/pipecg/sparse.py:43-132 (same
fields, coercion to int64/float64, same validation messages) so reference
code and tests construct it unchanged; reference ``CsrMatrix`` instances are
accepted anywhere by duck typing.  ``DeviceCsr`` is the B200 layout the
kernels read: int32 column indices (int32 or int64 row pointers), arrays
padded for the bulk-copy engine, uploaded once and cached on the matrix.
Stencil generators build matrices directly in HBM.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._device import cached_device, h2d_multi, host_fingerprint, require_cuda, stream_ptr

__all__ = [
    "CsrMatrix",
    "CapacityError",
    "csr_from_dense",
    "DeviceCsr",
    "as_device_csr",
    "stencil_shape",
    "stencil_device",
    "stencil_host",
    "poisson125_shape",
    "generate_poisson125",
    "generate_powerlaw",
    "MatrixMarketError",
    "parse_matrix_market",
    "load_matrix_market",
]

PAD = 16  # trailing elements the staged (bulk-copy) reads may touch


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input.  Carries the 1-based offending line
    (sparse.py:29-36: same message form ``line N: ...``)."""

    def __init__(self, message: str, line_number: int | None = None):
        self.line_number = line_number
        if line_number is not None:
            message = f"line {line_number}: {message}"
        super().__init__(message)


class CapacityError(RuntimeError):
    """Requested matrix would exceed the allowed memory budget (sparse.py:39-40)."""


@dataclass(frozen=True)
class CsrMatrix:
    """Compressed sparse row matrix with float64 values (sparse.py:43-132).

    Immutable after construction.  ``row_offsets`` has length ``n_rows + 1``
    with ``row_offsets[0] == 0`` and ``row_offsets[-1] == nnz``; column
    indices are 0-based and strictly increasing within each row.
    """

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "n_rows", int(self.n_rows))
        object.__setattr__(self, "n_cols", int(self.n_cols))
        object.__setattr__(self, "row_offsets", np.ascontiguousarray(self.row_offsets, dtype=np.int64))
        object.__setattr__(self, "col_indices", np.ascontiguousarray(self.col_indices, dtype=np.int64))
        object.__setattr__(self, "values", np.ascontiguousarray(self.values, dtype=np.float64))
        self._validate()

    def _validate(self):
        # sparse.py:73-99 (host-side input validation, not part of the solve)
        if self.n_rows < 0 or self.n_cols < 0:
            raise ValueError("matrix dimensions must be nonnegative")
        ro = self.row_offsets
        if ro.ndim != 1 or ro.shape[0] != self.n_rows + 1:
            raise ValueError("row_offsets must have length n_rows + 1")
        if ro[0] != 0:
            raise ValueError("row_offsets must start at 0")
        if np.any(np.diff(ro) < 0):
            raise ValueError("row_offsets must be nondecreasing")
        nnz = int(ro[-1])
        if self.col_indices.shape != (nnz,) or self.values.shape != (nnz,):
            raise ValueError("col_indices/values length must equal row_offsets[-1]")
        if nnz:
            ci = self.col_indices
            if ci.min() < 0 or ci.max() >= self.n_cols:
                raise ValueError("column index out of range")
            d = np.diff(ci)
            if d.size:
                mask = np.ones(d.size, dtype=bool)
                bound = ro[1:-1]
                bound = bound[(bound > 0) & (bound < nnz)]
                mask[bound - 1] = False
                if np.any(d[mask] <= 0):
                    raise ValueError("column indices must be strictly increasing within a row")

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def row_length(self, i: int) -> int:
        return int(self.row_offsets[i + 1] - self.row_offsets[i])

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def take_rows(self, count: int) -> "CsrMatrix":
        count = max(0, min(int(count), self.n_rows))
        end = int(self.row_offsets[count])
        return CsrMatrix(count, self.n_cols, self.row_offsets[: count + 1].copy(),
                         self.col_indices[:end].copy(), self.values[:end].copy())

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        row_ids = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        out[row_ids, self.col_indices] = self.values
        return out

    def to_device(self) -> "DeviceCsr":
        return as_device_csr(self)


def csr_from_dense(dense) -> CsrMatrix:
    """Build a CsrMatrix from a 2-D array, dropping exact zeros (sparse.py:172-181)."""
    dense = np.asarray(dense, dtype=np.float64)
    if dense.ndim != 2:
        raise ValueError("expected a 2-D array")
    n_rows, n_cols = dense.shape
    rows, cols = np.nonzero(dense)
    row_offsets = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=row_offsets[1:])
    return CsrMatrix(n_rows, n_cols, row_offsets, cols.astype(np.int64), dense[rows, cols])


@dataclass
class DeviceCsr:
    """A CSR matrix resident in HBM in the kernels' layout.

    rowptr: int32 (nnz < 2^31) or int64, length n_rows + 1 + PAD (padded with
    nnz); col: int32, length nnz + PAD; val: float64, length nnz + PAD.
    """

    n_rows: int
    n_cols: int
    nnz: int
    rowptr: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor
    host: object = None  # the CsrMatrix it came from, if any
    _long_rows: torch.Tensor | None = field(default=None, repr=False)
    _n_long: int = -1

    @property
    def rp64(self) -> int:
        return 1 if self.rowptr.dtype == torch.int64 else 0

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def long_rows(self) -> tuple[int, int]:
        """(device pointer, count) of rows longer than the thread-per-row limit."""
        if self._n_long < 0:
            cnt = ctypes.c_int64(0)
            _lib.call("pipecg_b200_find_long_rows", self.n_rows, self.rp64, self.rowptr.data_ptr(),
                      256, None, 0, ctypes.byref(cnt), stream_ptr())
            n = int(cnt.value)
            if n:
                lr = torch.empty(n, dtype=torch.int32, device=self.col.device)
                _lib.call("pipecg_b200_find_long_rows", self.n_rows, self.rp64,
                          self.rowptr.data_ptr(), 256, lr.data_ptr(), n, ctypes.byref(cnt),
                          stream_ptr())
                self._long_rows = lr
            self._n_long = n
        return (self._long_rows.data_ptr() if self._long_rows is not None else None, self._n_long)

    def row_patterns(self, codes: bool = False):
        """The matrix's lossless row-pattern dictionary (what fused variants
        E/F read instead of the CSR): (number of distinct rows up to the row
        index shift, dictionary entries[, uint8 code per row]).  (0, 0) when
        the rows are too diverse for a dictionary."""
        n_pat, n_e = ctypes.c_int64(0), ctypes.c_int64(0)
        out = torch.empty(self.n_rows, dtype=torch.uint8, device=self.col.device) if codes else None
        _lib.call("pipecg_b200_row_patterns", self.n_rows, self.rp64, self.rowptr.data_ptr(),
                  self.col.data_ptr(), self.val.data_ptr(), ctypes.byref(n_pat), ctypes.byref(n_e),
                  out.data_ptr() if out is not None else None, stream_ptr())
        if codes:
            return int(n_pat.value), int(n_e.value), (out if n_pat.value else None)
        return int(n_pat.value), int(n_e.value)

    def to_host(self) -> CsrMatrix:
        ro = self.rowptr[: self.n_rows + 1].to(torch.int64).cpu().numpy()
        ci = self.col[: self.nnz].to(torch.int64).cpu().numpy()
        va = self.val[: self.nnz].cpu().numpy()
        return CsrMatrix(self.n_rows, self.n_cols, ro, ci, va)


def _narrow(src: torch.Tensor, dst: torch.Tensor) -> None:
    ovf = ctypes.c_int(0)
    _lib.call("pipecg_b200_narrow_i64", src.numel(), src.data_ptr(), dst.data_ptr(),
              ctypes.byref(ovf), stream_ptr())


def upload_csr(A) -> DeviceCsr:
    """Upload any CsrMatrix-like object (duck-typed: n_rows, n_cols,
    row_offsets, col_indices, values) into the device layout."""
    dev = require_cuda()
    n, m = int(A.n_rows), int(A.n_cols)
    ro = np.ascontiguousarray(A.row_offsets, dtype=np.int64)
    nnz = int(ro[-1]) if ro.size else 0
    if m >= 2**31:
        raise ValueError("matrices with >= 2^31 columns must be sharded across devices")
    rp64 = nnz >= 2**31
    # host-side narrowing in the native pinned pipeline (csrc/hostio.cu):
    # 12 bytes per nonzero cross PCIe instead of the host layout's 16
    rowptr = torch.empty(n + 1 + PAD, dtype=torch.int64 if rp64 else torch.int32, device=dev)
    rowptr[n + 1:].fill_(nnz)
    col = torch.empty(nnz + PAD, dtype=torch.int32, device=dev)
    val = torch.empty(nnz + PAD, dtype=torch.float64, device=dev)
    col[nnz:].zero_()
    val[nnz:].zero_()
    # one interleaved pass: the column narrowing (host-bound) overlaps the
    # value copies (PCIe-bound)
    items = [(rowptr[: n + 1], ro, not rp64)]
    if nnz:
        items += [(col[:nnz], np.ascontiguousarray(A.col_indices, dtype=np.int64), True),
                  (val[:nnz], np.ascontiguousarray(A.values, dtype=np.float64), False)]
    h2d_multi(items)
    return DeviceCsr(n, m, nnz, rowptr, col, val, host=A)


def as_device_csr(A) -> DeviceCsr:
    """Device form of ``A`` (uploaded once and cached on the object)."""
    if isinstance(A, DeviceCsr):
        return A
    return cached_device(A, "_b200_device", lambda: upload_csr(A), A.row_offsets, A.col_indices,
                         A.values)


# --- stencil generators (device) -------------------------------------------

_KINDS = {"2d5": 5, "3d7": 7, "3d27": 27, "p125": 125, 5: 5, 7: 7, 27: 27, 125: 125}


def stencil_shape(kind, n: int) -> tuple[int, int]:
    """(N, nnz) of a stencil matrix: kind 2d5 / 3d7 / 3d27 / p125."""
    k = _KINDS[kind]
    N, nnz = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("pipecg_b200_stencil_shape", k, int(n), ctypes.byref(N), ctypes.byref(nnz))
    return int(N.value), int(nnz.value)


def stencil_device(kind, n: int, row_begin: int = 0, row_end: int | None = None) -> DeviceCsr:
    """Generate (a row block of) a stencil matrix directly in HBM.

    Natural x-fastest ordering, ascending columns; values as the reference /
    SURVEY.md §8(d): 2D 5-pt diag 4, 3D 7-pt diag 6, 3D 27-pt diag 26 (all
    26 neighbours -1), 125-pt diag = entry count (kernels.py:35-61).
    """
    dev = require_cuda()
    k = _KINDS[kind]
    N, _ = stencil_shape(k, n)
    row_end = N if row_end is None else int(row_end)
    rows = row_end - row_begin
    lo = _prefix_count(k, n, row_begin)
    hi = _prefix_count(k, n, row_end)
    nnz = hi - lo
    rp64 = nnz >= 2**31
    rowptr = torch.empty(rows + 1 + PAD, dtype=torch.int64 if rp64 else torch.int32, device=dev)
    col = torch.zeros(nnz + PAD, dtype=torch.int32, device=dev)
    val = torch.zeros(nnz + PAD, dtype=torch.float64, device=dev)
    _lib.call("pipecg_b200_stencil_fill", k, int(n), int(row_begin), int(row_end), int(rp64),
              rowptr.data_ptr(), col.data_ptr(), val.data_ptr(), stream_ptr())
    rowptr[rows + 1:].fill_(nnz)
    return DeviceCsr(rows, N, nnz, rowptr, col, val)


def _prefix_count(k: int, n: int, row: int) -> int:
    """Entries in rows [0, row) (closed form evaluated by generators.cu)."""
    out = ctypes.c_int64()
    _lib.call("pipecg_b200_stencil_prefix", k, int(n), int(row), ctypes.byref(out))
    return int(out.value)


def stencil_host(kind, n: int) -> CsrMatrix:
    """Stencil matrix generated on the device and returned as a host CsrMatrix."""
    d = stencil_device(kind, n)
    A = d.to_host()
    object.__setattr__(A, "_b200_device",
                       (d, host_fingerprint(A.row_offsets, A.col_indices, A.values)))
    return A


def poisson125_shape(n: int) -> tuple[int, int]:
    """Closed-form (N, nnz) of the order-n 125-point stencil (sparse.py:329-340)."""
    n = int(n)
    if n < 5:
        raise ValueError("stencil requires n >= 5")
    return n**3, (5 * n - 6) ** 3


def generate_poisson125(n: int, max_bytes: int = 2**31) -> CsrMatrix:
    """The reference's 125-point test matrix (sparse.py:347-375), generated
    on the device.  Same CapacityError budget as the reference."""
    N, nnz = poisson125_shape(n)
    need = 16 * nnz + 8 * (N + 1)
    if need > max_bytes:
        raise CapacityError(
            f"n={n} needs about {need / 2**30:.2f} GiB (budget {max_bytes / 2**30:.2f} GiB)"
        )
    return stencil_host("p125", n)


def generate_powerlaw(n_rows: int = 2**22, seed: int = 20261017, tau: float = 2.2,
                      avg_degree: float = 11.92) -> CsrMatrix:
    """BASELINE.json configs[3]: irregular SPD CSR with power-law row lengths.

    The recipe of SURVEY.md §8(d) config 4 (host numpy; it is defined by
    numpy's PCG64 stream): weights w_i = (i+10)^(-1/(tau-1)); M =
    (avg_degree*N - N)/2 edges, one endpoint drawn with probability
    proportional to w, the other uniform; self-loops dropped; values
    -U(0.1, 1.0), duplicates summed per unordered pair then mirrored
    (exactly symmetric); diagonal =
    sum |offdiag| + 1 (strictly diagonally dominant, hence SPD).  At the
    default N = 2^22 this gives nnz = 49,986,874 and row lengths 1 .. 49,349
    (median 9), the figures SURVEY.md records.
    """
    N = int(n_rows)
    rng = np.random.default_rng(seed)
    w = (np.arange(N) + 10.0) ** (-1.0 / (tau - 1.0))
    M = int((avg_degree * N - N) / 2)
    src = rng.choice(N, size=M, p=w / w.sum())
    dst = rng.integers(0, N, size=M)
    vals = -rng.uniform(0.1, 1.0, size=M)
    keep = src != dst
    src, dst, vals = src[keep], dst[keep], vals[keep]
    # duplicates summed once per unordered pair (draw order), then mirrored:
    # the matrix is exactly symmetric
    lo, hi = np.minimum(src, dst), np.maximum(src, dst)
    key = lo * N + hi
    order = np.argsort(key, kind="stable")
    key = key[order]
    v = vals[order]
    first = np.ones(key.size, dtype=bool)
    first[1:] = key[1:] != key[:-1]
    starts = np.flatnonzero(first)
    pk = key[starts]
    pv = np.add.reduceat(v, starts) if v.size else v
    a, b = pk // N, pk % N
    r = np.concatenate([a, b])
    c = np.concatenate([b, a])
    uv = np.concatenate([pv, pv])
    order = np.argsort(r * N + c, kind="stable")
    ur, uc, uv = r[order], c[order], uv[order]
    diag = np.bincount(ur, weights=np.abs(uv), minlength=N) + 1.0
    # merge the diagonal into ascending column order per row
    counts = np.bincount(ur, minlength=N) + 1
    row_offsets = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(counts, out=row_offsets[1:])
    nnz = int(row_offsets[-1])
    below = np.bincount(ur[uc < ur], minlength=N)  # entries left of the diagonal
    dpos = row_offsets[:-1] + below
    is_diag = np.zeros(nnz, dtype=bool)
    is_diag[dpos] = True
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    col[dpos] = np.arange(N)
    val[dpos] = diag
    col[~is_diag] = uc
    val[~is_diag] = uv
    return CsrMatrix(N, N, row_offsets, col, val)


# --- Matrix Market ingestion ---------------------------

def _mm_raise(rc: int) -> None:
    msg = _lib.last_error()
    suffix = f" (code {rc})"
    if msg.endswith(suffix):
        msg = msg[: -len(suffix)]
    if rc == _lib.PCG_EPARSE:
        line = int(_lib.load().pipecg_b200_mm_error_line())
        prefix = f"line {line}: "
        raise MatrixMarketError(msg[len(prefix):] if msg.startswith(prefix) else msg, line)
    if rc == _lib.PCG_EIO:
        raise OSError(msg)
    raise _lib.NativeError("Matrix Market ingestion", rc, msg)


def _mm_csr(handle) -> CsrMatrix:
    """COO handle -> CSR built on the device; returns the host CsrMatrix (the
    reference's return type) with the device copy cached on it."""
    L = _lib.load()
    try:
        n_rows, n_cols, n_coo = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.call("pipecg_b200_mm_info", handle, ctypes.byref(n_rows), ctypes.byref(n_cols),
                  ctypes.byref(n_coo))
        n, m, cap = int(n_rows.value), int(n_cols.value), int(n_coo.value)
        dev = require_cuda()
        rp64 = cap >= 2**31
        rowptr = torch.empty(n + 1 + PAD, dtype=torch.int64 if rp64 else torch.int32, device=dev)
        col = torch.zeros(cap + PAD, dtype=torch.int32, device=dev)
        val = torch.zeros(cap + PAD, dtype=torch.float64, device=dev)
        nnz = ctypes.c_int64()
        rc = L.pipecg_b200_mm_to_csr(handle, int(rp64), rowptr.data_ptr(), col.data_ptr(),
                                     val.data_ptr(), ctypes.byref(nnz), stream_ptr())
        if rc:
            _mm_raise(rc)
    finally:
        L.pipecg_b200_mm_free(handle)
    rowptr[n + 1:].fill_(int(nnz.value))
    d = DeviceCsr(n, m, int(nnz.value), rowptr, col, val)
    A = d.to_host()
    object.__setattr__(A, "_b200_device",
                       (d, host_fingerprint(A.row_offsets, A.col_indices, A.values)))
    return A


def parse_matrix_market(source) -> CsrMatrix:
    """Parse a Matrix Market coordinate document (sparse.py:195-320).

    ``source`` is the document text or an open text stream.  Only
    ``matrix coordinate real general|symmetric`` is accepted; symmetric
    storage is mirrored, duplicate coordinates are summed (document order);
    malformed input raises :class:`MatrixMarketError` naming the 1-based
    line, exactly as the reference does.  Tokenising runs in the native
    multi-threaded parser (csrc/mmio.cu); the CSR is assembled on the GPU."""
    text = source if isinstance(source, str) else source.read()
    data = text.encode("utf-8", errors="replace")
    h = ctypes.c_void_p()
    rc = _lib.load().pipecg_b200_mm_parse(data, len(data), 0, ctypes.byref(h))
    if rc:
        _mm_raise(rc)
    return _mm_csr(h)


def load_matrix_market(path) -> CsrMatrix:
    """Read and parse a Matrix Market file (sparse.py:323-326; universal
    newlines like the reference's text-mode read)."""
    import os

    h = ctypes.c_void_p()
    rc = _lib.load().pipecg_b200_mm_read(os.fsencode(path), ctypes.byref(h))
    if rc:
        _mm_raise(rc)
    return _mm_csr(h)
