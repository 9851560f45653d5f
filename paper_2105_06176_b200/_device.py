"""Device plumbing: torch CUDA tensors as the memory of the C-ABI kernels.

PyTorch is used only for device memory, streams and host<->device copies;
all arithmetic on the solve path runs in the sm_100a kernels of
``_lib/libpipecg_b200.so``.
"""

from __future__ import annotations

import numpy as np
import torch

_F64 = torch.float64


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2105_06176_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback"
        )
    return torch.device("cuda", torch.cuda.current_device())


def shared_max_sms(ranks_on_device: int, device: int | None = None) -> int:
    """``DeviceOptions.max_sms`` for one of ``ranks_on_device`` solvers that
    share a GPU: the device's SM count split between them (less a margin),
    so every rank's persistent grid stays co-resident while its prologue
    waits for the peers."""
    k = max(1, int(ranks_on_device))
    if k == 1:
        return 0
    dev = torch.cuda.current_device() if device is None else int(device)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    return max(8, sms // k - 10)


def host_fingerprint(*arrays, samples: int = 2048) -> tuple:
    """Cheap content fingerprint of host arrays for the device-copy caches:
    each array's identity (data pointer, shape, dtype) and a hash of a
    strided sample of its bytes (``samples`` elements + the last one, tens
    of microseconds whatever the size).

    The reference's CsrMatrix and JacobiPreconditioner are immutable after
    construction (sparse.py:43-50, kernels.py:204); a caller that rewrites
    their arrays in place anyway gets a fresh upload when the sample
    changes.  A change that misses every sampled element is not detected:
    call :func:`invalidate_device_cache` after such an edit."""
    out = []
    for a in arrays:
        a = np.asarray(a)
        flat = a.reshape(-1)
        n = flat.size
        h = 0
        if n:
            step = max(1, n // samples)
            h = hash(flat[::step].tobytes()) ^ hash(flat[-1:].tobytes())
        out.append((a.__array_interface__["data"][0], a.shape, a.dtype.str, h))
    return tuple(out)


def cached_device(owner, attr: str, make, *host_arrays):
    """``owner.attr`` holds (device copy, fingerprint of ``host_arrays``);
    the copy is rebuilt with ``make()`` when the fingerprint changed or the
    copy lives on another device."""
    fp = host_fingerprint(*host_arrays)
    hit = getattr(owner, attr, None)
    if isinstance(hit, tuple) and len(hit) == 2 and hit[1] == fp and _on_current(hit[0]):
        return hit[0]
    d = make()
    try:
        object.__setattr__(owner, attr, (d, fp))
    except (AttributeError, TypeError):
        pass
    return d


def _on_current(d) -> bool:
    t = d if isinstance(d, torch.Tensor) else getattr(d, "col", None)
    return isinstance(t, torch.Tensor) and t.device.index == torch.cuda.current_device()


def invalidate_device_cache(obj) -> None:
    """Forget the device copy (and the solvers built on it) cached on a
    host CsrMatrix or JacobiPreconditioner -- after an in-place edit of its
    arrays, which the reference's contract forbids (immutable objects) and
    the sampled fingerprint may miss."""
    for attr in ("_b200_device", "_b200_inv_diag"):
        if attr in getattr(obj, "__dict__", {}):
            try:
                object.__delattr__(obj, attr)
            except AttributeError:
                pass


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def is_device_tensor(v) -> bool:
    return isinstance(v, torch.Tensor) and v.is_cuda


def host_f64(v) -> np.ndarray:
    """Reference coercion (kernels.py:145-149): contiguous float64 ndarray."""
    if isinstance(v, torch.Tensor):
        v = v.detach().cpu().numpy()
    return np.ascontiguousarray(v, dtype=np.float64)


def to_device_f64(v, pad: int = 0) -> torch.Tensor:
    """Copy a host vector (or reuse a CUDA float64 tensor) on the device."""
    dev = require_cuda()
    if is_device_tensor(v):
        t = v if v.dtype == _F64 else v.to(_F64)
        t = t.contiguous()
        if pad:
            out = torch.zeros(t.numel() + pad, dtype=_F64, device=t.device)
            out[: t.numel()].copy_(t)
            return out
        return t
    a = host_f64(v).reshape(-1)
    out = torch.empty(a.size + pad, dtype=_F64, device=dev)
    if pad:
        out[a.size:].zero_()
    if a.size:
        h2d(out, a)
    return out


def h2d(dst: torch.Tensor, src: np.ndarray, narrow: bool = False) -> None:
    """Host -> device through the native pinned pipeline (csrc/hostio.cu).

    ``src`` is a contiguous int64 / float64 host array; with ``narrow`` the
    int64 values are narrowed to the int32 ``dst`` on the host side."""
    from . import _lib

    src = np.ascontiguousarray(src)
    kind = _lib.PCG_H2D_I64_TO_I32 if narrow else _lib.PCG_H2D_COPY64
    _lib.call("pipecg_b200_h2d", dst.data_ptr(), src.ctypes.data, src.size, kind, stream_ptr())
    # the staging ring is reused by the next transfer; the caller's stream
    # orders the copies before any kernel that reads dst


def h2d_multi(items) -> None:
    """Several host -> device transfers in one pass of the pinned pipeline,
    their chunks interleaved (host-bound narrowing overlaps PCIe-bound
    copies).  ``items``: (dst tensor, contiguous int64 / float64 host array,
    narrow) triples, as for :func:`h2d`."""
    import ctypes

    from . import _lib

    items = [(d, np.ascontiguousarray(a), bool(nw)) for d, a, nw in items if np.asarray(a).size]
    k = len(items)
    if not k:
        return
    dst = (ctypes.c_void_p * k)(*[d.data_ptr() for d, _, _ in items])
    src = (ctypes.c_void_p * k)(*[a.ctypes.data for _, a, _ in items])
    cnt = (ctypes.c_int64 * k)(*[a.size for _, a, _ in items])
    kinds = (ctypes.c_int * k)(*[_lib.PCG_H2D_I64_TO_I32 if nw else _lib.PCG_H2D_COPY64
                                 for _, _, nw in items])
    _lib.call("pipecg_b200_h2d_multi", k, dst, src, cnt, kinds, stream_ptr())


def d2h(src: torch.Tensor) -> np.ndarray:
    """Device float64 vector -> new host ndarray (native pinned pipeline)."""
    from . import _lib

    src = src.contiguous()
    out = np.empty(src.numel(), dtype=np.float64)
    if out.size:
        _lib.call("pipecg_b200_d2h", out.ctypes.data, src.data_ptr(), out.nbytes, stream_ptr())
    return out


def vec_len(v) -> int:
    if isinstance(v, torch.Tensor):
        return v.numel() if v.dim() == 1 else -1
    a = np.asarray(v)
    return a.size if a.ndim == 1 else -1


def warm_transfers() -> None:
    """Allocate the pinned staging ring and start the host thread pool of the
    transfer pipeline (one-time per process; otherwise the first upload
    pays for it)."""
    t = torch.empty(1, dtype=_F64, device=require_cuda())
    h2d(t, np.zeros(1))
    d2h(t)
