"""The reference's operator surface (kernels.py) on B200 kernels.

Same names, argument meaning and errors as
/root/reference/pkg/src/pipecg/kernels.py:152-267.  Every function accepts
numpy arrays (copied to HBM, result copied back, ``out=`` honoured like the
reference) or CUDA ``torch`` tensors (computed in place on the device, on
the current torch stream).  All arithmetic runs in the sm_100a kernels of
``_lib/libpipecg_b200.so``; there is no CPU fallback.

Bitwise contract (kernels.py:1-7): spmv, jacobi_apply and
fused_pipecg_update round exactly like the reference (no FMA, CSR order);
``dot`` defaults to the reference's strict left-to-right order
(``mode="seq"``, one warp); ``mode="tree"`` is the deterministic parallel
reduction the solver uses.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import (cached_device, host_f64, host_fingerprint, is_device_tensor, require_cuda,
                      stream_ptr, to_device_f64,
                      vec_len)
from .sparse import DeviceCsr, as_device_csr

__all__ = [
    "spmv",
    "residual",
    "dot",
    "dots",
    "norm2",
    "JacobiPreconditioner",
    "jacobi_setup",
    "jacobi_apply",
    "fused_pipecg_update",
    "fused_pipecg_update_pc_dots",
]

_DOT_MODES = {"seq": _lib.PCG_DOT_SEQ, "tree": _lib.PCG_DOT_TREE}


def _check_len(v, length: int, name: str) -> None:
    # kernels.py:145-149 (_as_vector)
    if vec_len(v) != length:
        raise ValueError(f"{name} must be a vector of length {length}")


def _host_out(out, length: int, name: str) -> np.ndarray:
    _check_len(out, length, name)
    return np.ascontiguousarray(out, dtype=np.float64)


def _finish_host(result_dev: torch.Tensor, out, length: int) -> np.ndarray:
    """Copy a device result into a host out= array (or a new array)."""
    host = result_dev[:length].cpu().numpy()
    if out is None:
        return host.copy()
    dst = np.ascontiguousarray(out, dtype=np.float64)
    dst[...] = host
    return dst


def spmv(matrix, x, out=None):
    """Sparse matrix-vector product ``out = matrix @ x`` (kernels.py:152-164).

    Rows accumulate left to right in storage order (bitwise equal to the
    reference for rows of <= 256 entries; longer rows use a deterministic
    block tree)."""
    A = as_device_csr(matrix)
    _check_len(x, A.n_cols, "x")
    if out is not None:
        _check_len(out, A.n_rows, "out")
    lr, nl = A.long_rows()
    if is_device_tensor(x):
        xd = to_device_f64(x)
        y = out if is_device_tensor(out) and out.dtype == torch.float64 and out.is_contiguous() \
            else torch.empty(A.n_rows, dtype=torch.float64, device=xd.device)
        _lib.call("pipecg_b200_spmv", A.n_rows, A.rp64, A.rowptr.data_ptr(), A.col.data_ptr(),
                  A.val.data_ptr(), xd.data_ptr(), y.data_ptr(), lr, nl, stream_ptr())
        if out is not None and y is not out:
            out.copy_(y)
            return out
        return y
    xd = to_device_f64(x)
    y = torch.empty(max(A.n_rows, 1), dtype=torch.float64, device=xd.device)
    _lib.call("pipecg_b200_spmv", A.n_rows, A.rp64, A.rowptr.data_ptr(), A.col.data_ptr(),
              A.val.data_ptr(), xd.data_ptr(), y.data_ptr(), lr, nl, stream_ptr())
    return _finish_host(y, out, A.n_rows)


def residual(matrix, x, b):
    """b - matrix @ x with the reference's two roundings (solvers.py:307)."""
    A = as_device_csr(matrix)
    _check_len(x, A.n_cols, "x")
    _check_len(b, A.n_rows, "b")
    lr, nl = A.long_rows()
    xd, bd = to_device_f64(x), to_device_f64(b)
    r = torch.empty(max(A.n_rows, 1), dtype=torch.float64, device=xd.device)
    _lib.call("pipecg_b200_residual", A.n_rows, A.rp64, A.rowptr.data_ptr(), A.col.data_ptr(),
              A.val.data_ptr(), xd.data_ptr(), bd.data_ptr(), r.data_ptr(), lr, nl, stream_ptr())
    if is_device_tensor(x) or is_device_tensor(b):
        return r[: A.n_rows]
    return r[: A.n_rows].cpu().numpy()


_WS = {}


def _dots_workspace(dev) -> torch.Tensor:
    key = dev.index
    ws = _WS.get(key)
    if ws is None:
        nbytes = int(_lib.load().pipecg_b200_dots_workspace_bytes())
        ws = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
        _WS[key] = ws
    return ws


def dots(pairs, mode: str = "seq") -> list[float]:
    """Up to four dot products in one pass over HBM: [(a0, b0), (a1, b1), ...]."""
    require_cuda()
    if not 1 <= len(pairs) <= 4:
        raise ValueError("dots takes 1 to 4 pairs")
    n = vec_len(pairs[0][0])
    dev_vecs = []
    for a, b in pairs:
        if vec_len(a) < 0:
            raise ValueError("a must be a vector")
        _check_len(a, n, "a")
        _check_len(b, n, "b")
        dev_vecs.append((to_device_f64(a), to_device_f64(b)))
    dev = dev_vecs[0][0].device
    out = torch.empty(4, dtype=torch.float64, device=dev)
    A = (ctypes.c_void_p * 4)(*[p[0].data_ptr() for p in dev_vecs] + [0] * (4 - len(pairs)))
    B = (ctypes.c_void_p * 4)(*[p[1].data_ptr() for p in dev_vecs] + [0] * (4 - len(pairs)))
    _lib.call("pipecg_b200_dots", n, len(pairs), ctypes.cast(A, ctypes.c_void_p),
              ctypes.cast(B, ctypes.c_void_p), _DOT_MODES[mode], out.data_ptr(),
              _dots_workspace(dev).data_ptr(), stream_ptr())
    return [float(v) for v in out[: len(pairs)].cpu().tolist()]


def dot(a, b, mode: str = "seq") -> float:
    """Inner product (kernels.py:192-196).  ``mode="seq"`` is the reference's
    strict left-to-right accumulation (bitwise); ``"tree"`` is the fast
    deterministic block reduction."""
    n = vec_len(a)
    if n < 0:
        a = host_f64(a).reshape(-1)
        n = a.size
    _check_len(b, n, "b")
    return dots([(a, b)], mode)[0]


def norm2(a, mode: str = "seq") -> float:
    """Euclidean norm built on :func:`dot` (kernels.py:199-201)."""
    return float(np.sqrt(dot(a, a, mode)))


@dataclass(frozen=True)
class JacobiPreconditioner:
    """Reciprocal diagonal of a matrix, applied elementwise (kernels.py:204-215).

    ``inv_diag`` is a host ndarray or a CUDA tensor; the device copy used by
    the kernels is cached on the object."""

    inv_diag: object

    @property
    def n(self) -> int:
        return int(self.inv_diag.numel() if isinstance(self.inv_diag, torch.Tensor)
                   else np.asarray(self.inv_diag).size)

    def take(self, start: int, stop: int) -> "JacobiPreconditioner":
        return JacobiPreconditioner(self.inv_diag[start:stop].clone()
                                    if isinstance(self.inv_diag, torch.Tensor)
                                    else np.asarray(self.inv_diag)[start:stop].copy())


def device_inv_diag(pc) -> torch.Tensor:
    """Device float64 copy of ``pc.inv_diag`` (cached on the object)."""
    if is_device_tensor(pc.inv_diag):
        return to_device_f64(pc.inv_diag)  # the caller's device tensor: no copy to go stale
    return cached_device(pc, "_b200_inv_diag", lambda: to_device_f64(pc.inv_diag), pc.inv_diag)


def jacobi_setup(matrix) -> JacobiPreconditioner:
    """Extract the diagonal and invert it on the device (kernels.py:218-237).

    Raises ``ValueError`` naming the first row whose diagonal entry is
    missing (checked first, as the reference) or exactly zero."""
    if int(matrix.n_rows) != int(matrix.n_cols):
        raise ValueError("diagonal preconditioner needs a square matrix")
    A = as_device_csr(matrix)
    d = torch.empty(max(A.n_rows, 1), dtype=torch.float64, device=A.val.device)
    bad_row, bad_kind = ctypes.c_int64(-1), ctypes.c_int(0)
    rc = _lib.load().pipecg_b200_jacobi_setup(A.n_rows, A.rp64, A.rowptr.data_ptr(),
                                              A.col.data_ptr(), A.val.data_ptr(), d.data_ptr(),
                                              ctypes.byref(bad_row), ctypes.byref(bad_kind),
                                              stream_ptr())
    if rc == _lib.PCG_EDIAG:
        what = "missing diagonal entry" if bad_kind.value == 1 else "zero diagonal entry"
        raise ValueError(f"row {bad_row.value}: {what}")
    _lib.check("pipecg_b200_jacobi_setup", rc)
    d = d[: A.n_rows]
    if isinstance(matrix, DeviceCsr):
        return JacobiPreconditioner(d)
    pc = JacobiPreconditioner(d.cpu().numpy())
    object.__setattr__(pc, "_b200_inv_diag", (d, host_fingerprint(pc.inv_diag)))
    return pc


def jacobi_apply(pc, v, out=None):
    """out = inv_diag * v (kernels.py:240-247)."""
    n = pc.n
    _check_len(v, n, "v")
    if out is not None:
        _check_len(out, n, "out")
    d = device_inv_diag(pc)
    vd = to_device_f64(v)
    if is_device_tensor(out) and out.dtype == torch.float64 and out.is_contiguous():
        res = out
    else:
        res = torch.empty(max(n, 1), dtype=torch.float64, device=d.device)
    _lib.call("pipecg_b200_jacobi_apply", n, d.data_ptr(), vd.data_ptr(), res.data_ptr(),
              stream_ptr())
    if is_device_tensor(v) or is_device_tensor(out):
        if out is not None and res is not out:
            out.copy_(res[:n])
            return out
        return res[:n] if res is not out else out
    return _finish_host(res, out, n)


_LANES = ("z", "q", "s", "p", "x", "r", "u", "w")


def fused_pipecg_update(state, alpha: float, beta: float) -> None:
    """All eight pipelined-CG recurrences in one pass (kernels.py:250-267).

    ``state`` is any object carrying the ten vectors z, q, s, p, x, r, u, w,
    m, n as attributes; the first eight are updated in place (numpy arrays
    are round-tripped through HBM)."""
    names = _LANES + ("m", "n")
    vecs = [getattr(state, k) for k in names]
    n = vec_len(vecs[4])
    for k, v in zip(names, vecs):
        _check_len(v, n, k)
    dev = require_cuda()
    on_device = all(is_device_tensor(v) and v.dtype == torch.float64 and v.is_contiguous()
                    for v in vecs)
    if on_device:
        d = vecs
    else:
        d = [to_device_f64(v) for v in vecs]
    _lib.call("pipecg_b200_fused_update", n, *[t.data_ptr() for t in d], float(alpha),
              float(beta), stream_ptr())
    if not on_device:
        for k, src, dv in zip(names[:8], vecs[:8], d[:8]):
            host = dv.cpu().numpy() if dv.numel() else np.empty(0)
            if isinstance(src, np.ndarray) and src.dtype == np.float64 and src.flags.c_contiguous:
                src[...] = host
            elif isinstance(src, torch.Tensor):
                src.copy_(dv)
            else:
                setattr(state, k, host.copy())
    del dev


def fused_pipecg_update_pc_dots(state, inv_diag, alpha: float, beta: float,
                                mode: str = "tree") -> tuple[float, float, float]:
    """fused_pipecg_update + m = M^-1 w + (r,u), (w,u), (u,u) in one HBM pass
    (solvers.py:350-358 as one kernel).  Device tensors only."""
    names = _LANES + ("m", "n")
    vecs = [getattr(state, k) for k in names]
    if not all(is_device_tensor(v) for v in vecs):
        raise TypeError("fused_pipecg_update_pc_dots works on CUDA tensors")
    n = vecs[0].numel()
    d = to_device_f64(inv_diag)
    out = torch.empty(4, dtype=torch.float64, device=vecs[0].device)
    _lib.call("pipecg_b200_fused_update_pc_dots", n, *[t.data_ptr() for t in vecs], d.data_ptr(),
              float(alpha), float(beta), _DOT_MODES[mode], out.data_ptr(),
              _dots_workspace(out.device).data_ptr(), stream_ptr())
    g, dl, uu = out[:3].cpu().tolist()
    return g, dl, uu
