"""PIPECG (and PCG) drivers: the reference's solver API on B200.

Mirrors /root/reference/pkg/src/pipecg/solvers.py: ``SolverConfig``,
``SolverBreakdown``, ``PipecgState``, ``SolveReport``, ``pipecg_scalars``,
``pipecg_init``, ``pipecg_solve``, ``pcg_solve``, ``true_residual_norm`` --
same names, signatures, stopping rule (absolute tolerance on sqrt((u,u)),
strict ``<``), history/drift bookkeeping and breakdown precedence.

``pipecg_solve`` runs the whole iteration loop on the device
(csrc/solver.cu): one fused kernel per iteration, convergence decided on the
GPU, CUDA-graph chunks, one small host read per chunk.  Device-specific
choices live in :class:`DeviceOptions` (keyword-only), so the reference's
positional signature is untouched.
"""

from __future__ import annotations

import ctypes
import math
import threading
import time
from dataclasses import dataclass, field
from typing import Any

import numpy as np
import torch

from . import _lib
from ._device import is_device_tensor, require_cuda, stream_ptr, to_device_f64, vec_len
from .kernels import device_inv_diag, dot, dots, jacobi_apply, norm2, residual, spmv
from .sparse import as_device_csr

__all__ = [
    "SolverConfig",
    "SolverBreakdown",
    "PipecgState",
    "SolveReport",
    "DeviceOptions",
    "PipecgSolver",
    "pcg_solve",
    "pipecg_scalars",
    "pipecg_init",
    "pipecg_solve",
    "true_residual_norm",
]


@dataclass
class SolverConfig:
    """Iteration controls (solvers.py:36-58).

    ``tolerance`` is absolute and applies to the preconditioned residual
    norm sqrt((u, u)); ``drift_check_interval`` (0 = off) records
    |b - Ax - r| / |b| every k-th iteration.
    """

    tolerance: float = 1e-5
    max_iterations: int = 10000
    record_history: bool = False
    drift_check_interval: int = 0

    def __post_init__(self):
        if not self.tolerance > 0:
            raise ValueError("tolerance must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.drift_check_interval < 0:
            raise ValueError("drift_check_interval must be nonnegative")


class SolverBreakdown(RuntimeError):
    """A scalar left the representable/SPD regime mid-iteration (solvers.py:61-71)."""

    def __init__(self, quantity: str, iteration: int, value: float):
        self.quantity = quantity
        self.iteration = iteration
        self.value = value
        super().__init__(
            f"{quantity} = {value!r} at iteration {iteration}: "
            "input is not SPD or the recurrence lost finiteness"
        )


@dataclass
class PipecgState:
    """The ten iteration vectors and the scalar recurrence (solvers.py:74-101)."""

    x: Any
    r: Any
    u: Any
    w: Any
    m: Any
    n: Any
    z: Any
    q: Any
    s: Any
    p: Any
    gamma: float
    gamma_prev: float
    delta: float
    alpha: float
    alpha_prev: float
    beta: float
    norm: float
    iteration: int = 0


@dataclass
class SolveReport:
    """Outcome of one solver run (solvers.py:104-169)."""

    converged: bool
    iterations: int
    final_norm: float
    strategy: str
    history: list | None = None
    phase_times: dict = field(default_factory=dict)
    verification_error: float | None = None
    transfer_values: int = 0
    transfer_values_total: int = 0
    drift_history: list | None = None
    profile: Any = None
    partition: dict | None = None

    def to_dict(self) -> dict:
        return {
            "converged": bool(self.converged),
            "iterations": int(self.iterations),
            "final_norm": float(self.final_norm),
            "strategy": self.strategy,
            "history": None if self.history is None else [float(h) for h in self.history],
            "phase_times": {k: float(v) for k, v in self.phase_times.items()},
            "verification_error": None
            if self.verification_error is None
            else float(self.verification_error),
            "transfer_values": int(self.transfer_values),
            "transfer_values_total": int(self.transfer_values_total),
            "drift_history": None
            if self.drift_history is None
            else [[int(i), float(v)] for i, v in self.drift_history],
            "profile": None if self.profile is None else (
                self.profile.to_dict() if hasattr(self.profile, "to_dict") else dict(self.profile)),
            "partition": None if self.partition is None else dict(self.partition),
        }

    @classmethod
    def from_dict(cls, data: dict) -> "SolveReport":
        return cls(
            converged=data["converged"],
            iterations=data["iterations"],
            final_norm=data["final_norm"],
            strategy=data["strategy"],
            history=data.get("history"),
            phase_times=dict(data.get("phase_times", {})),
            verification_error=data.get("verification_error"),
            transfer_values=data.get("transfer_values", 0),
            transfer_values_total=data.get("transfer_values_total", 0),
            drift_history=data.get("drift_history"),
            profile=data.get("profile"),
            partition=data.get("partition"),
        )


@dataclass
class DeviceOptions:
    """B200 execution choices (not part of the reference API).

    dot_mode: "tree" (deterministic block reduction, default) or "seq" (the
      reference's left-to-right order: bitwise-identical histories).
    engine: "auto" (autotuned at solver creation for >= 1M rows), "fused"
      (one kernel per iteration; variant autotuned), "fused-a" / "fused-b" /
      "fused-c" / "fused-d" / "fused-p" (consumer gathers dinv*w / gather warps /
      stored m / nnz-balanced tiles with cooperative gathers, for irregular rows /
      C with a whole chunk of iterations in one persistent launch, for small
      latency-bound problems), "fused-e" / "fused-f" (A / C reading the
      matrix through its lossless row-pattern dictionary: one byte per row
      instead of the CSR, for constant-coefficient stencil-like matrices),
      "fused-g" (irregular rows: one SELL-C-sigma kernel per iteration, hub
      rows as nnz-bounded chunks inside it) or "two" (update kernel + SpMV
      kernel; general matrices, very long rows).
    chunk: iterations per CUDA-graph chunk (0 = sized from the problem).
    use_graphs: capture chunks as CUDA graphs.
    max_sms: size persistent grids for this many SMs (0 = all; used when
      several solvers must be co-resident on one GPU).
    """

    dot_mode: str = "tree"
    engine: str = "auto"
    chunk: int = 0
    use_graphs: bool = True
    max_sms: int = 0

    def native(self) -> _lib.PcgOptions:
        eng = {"auto": 0, "fused": 1, "two": 2, "fused-a": 3, "fused-b": 4,
               "fused-c": 5, "fused-d": 6, "fused-p": 7, "fused-e": 8,
               "fused-f": 9, "fused-g": 10, "pcg": 11}[self.engine]
        dm = {"tree": _lib.PCG_DOT_TREE, "seq": _lib.PCG_DOT_SEQ}[self.dot_mode]
        return _lib.PcgOptions(dm, eng, int(self.chunk), 1 if self.use_graphs else 0,
                               int(self.max_sms))

    def key(self) -> tuple:
        return (self.dot_mode, self.engine, int(self.chunk), bool(self.use_graphs),
                int(self.max_sms))


def _check_system(A, b, x0):
    """solvers.py:172-179 (shape checks; no data movement)."""
    if int(A.n_rows) != int(A.n_cols):
        raise ValueError("solvers need a square matrix")
    n = int(A.n_rows)
    if vec_len(b) != n or vec_len(x0) != n:
        raise ValueError("b and x0 must have length n_rows")


class PipecgSolver:
    """A native solver handle bound to one device matrix + preconditioner.

    Owns the state vectors (13 padded N-vectors in HBM) and the captured
    CUDA graphs; reused across solves on the same matrix."""

    def __init__(self, A, inv_diag: torch.Tensor, options: DeviceOptions | None = None):
        require_cuda()
        self.A = as_device_csr(A)
        self.options = options or DeviceOptions()
        self.inv_diag = inv_diag
        m = _lib.PcgMatrix(self.A.n_rows, self.A.n_cols, self.A.nnz, self.A.rp64,
                           self.A.rowptr.data_ptr(), self.A.col.data_ptr(), self.A.val.data_ptr(),
                           inv_diag.data_ptr())
        opts = self.options.native()
        h = ctypes.c_void_p()
        _lib.call("pipecg_b200_solver_create", ctypes.byref(m), ctypes.byref(opts), ctypes.byref(h))
        self._h = h
        self.n = self.A.n_rows
        self.lock = threading.Lock()  # held by the thread driving a solve

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().pipecg_b200_solver_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return _lib.load().pipecg_b200_solver_stream(self._h)

    def init(self, b: torch.Tensor, x0: torch.Tensor, tolerance: float, max_iterations: int,
             drift_check_interval: int = 0) -> None:
        self._b, self._x0 = b, x0  # keep alive while queued
        _lib.call("pipecg_b200_solver_init", self._h, b.data_ptr(), x0.data_ptr(), float(tolerance),
                  int(max_iterations), int(drift_check_interval), stream_ptr())

    def run(self, record_history: bool, max_iterations: int, drift_k: int):
        res = _lib.PcgResult()
        hist = np.empty(max_iterations + 1) if record_history else None
        nd = max_iterations // drift_k + 1 if drift_k > 0 else 0
        d_it = np.zeros(nd, dtype=np.int64) if nd else None
        d_val = np.zeros(nd) if nd else None
        _lib.call(
            "pipecg_b200_solver_run", self._h, ctypes.byref(res),
            None if hist is None else hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            0 if hist is None else hist.size,
            None if d_it is None else d_it.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            None if d_val is None else d_val.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            nd,
        )
        return res, hist, d_it, d_val

    def enqueue(self, count: int) -> None:
        _lib.call("pipecg_b200_solver_enqueue", self._h, int(count))

    def prepare(self, count: int) -> None:
        """Build the CUDA graphs a following enqueue(count) launches."""
        _lib.call("pipecg_b200_solver_prepare", self._h, int(count))

    def poll(self) -> _lib.PcgResult:
        res = _lib.PcgResult()
        _lib.call("pipecg_b200_solver_poll", self._h, ctypes.byref(res))
        return res

    def x_tensor(self) -> torch.Tensor:
        """A device tensor view-copy of the iterate x (length N)."""
        ptr = _lib.load().pipecg_b200_solver_x(self._h)
        out = torch.empty(self.n, dtype=torch.float64, device=self.A.val.device)
        torch.cuda.current_stream().synchronize()
        _cuda_memcpy_d2d(out.data_ptr(), ptr, self.n * 8)
        return out

    def x_host(self, out: np.ndarray | None = None) -> np.ndarray:
        """The iterate x downloaded into a new host array (or ``out``; native
        pinned pipeline, on the solver's stream)."""
        if out is None:
            out = np.empty(self.n, dtype=np.float64)
        if self.n:
            _lib.call("pipecg_b200_d2h", out.ctypes.data, _lib.load().pipecg_b200_solver_x(self._h),
                      self.n * 8, self.stream)
        return out

    def state_tensors(self) -> dict:
        ptrs = (ctypes.c_void_p * 10)()
        _lib.call("pipecg_b200_solver_state", self._h, ptrs)
        names = ("x", "r", "u", "w", "m", "n", "z", "q", "s", "p")
        out = {}
        for k, p in zip(names, ptrs):
            t = torch.empty(self.n, dtype=torch.float64, device=self.A.val.device)
            _cuda_memcpy_d2d(t.data_ptr(), p, self.n * 8)
            out[k] = t
        return out


def _cuda_memcpy_d2d(dst: int, src: int, nbytes: int) -> None:
    """Synchronous device-to-device copy between raw pointers."""
    # torch has no public "copy from raw pointer"; wrap the pointer as a
    # tensor through the CUDA array interface instead of calling cudart.
    class _Raw:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (p, False),
                                             "version": 3, "strides": None, "stream": None}

    n = nbytes // 8
    if n == 0:
        return
    s = torch.as_tensor(_Raw(src, n), device="cuda")
    d = torch.as_tensor(_Raw(dst, n), device="cuda")
    d.copy_(s)
    torch.cuda.current_stream().synchronize()


class _PrefaultedHost:
    """A new float64 host array whose pages host threads touch in the
    background while the GPU solves (``pipecg_b200_host_prefault``): the
    x download then runs at ~38 GB/s instead of the ~15 GB/s that the
    first-touch page faults of a fresh array allow."""

    def __init__(self, n: int):
        self.out = np.empty(n, dtype=np.float64)
        self._t = None
        if n:
            self._t = threading.Thread(target=_lib.call, daemon=True,
                                       args=("pipecg_b200_host_prefault", self.out.ctypes.data,
                                             self.out.nbytes))
            self._t.start()

    def get(self) -> np.ndarray:
        if self._t is not None:
            self._t.join()
        return self.out


_CACHE_LOCK = threading.Lock()


def _solver_for(A, pc, options: DeviceOptions) -> tuple[PipecgSolver, bool]:
    """A native solver for (matrix, preconditioner, options), LOCKED for the
    caller: ``(solver, cached)``.

    The matrix caches one solver (its state vectors and graphs stay resident
    across solves).  A solver handle is single-threaded state, so the caller
    holds ``solver.lock`` from init to the x download; a second thread
    solving the same matrix concurrently gets a private solver instead of
    sharing the busy one (the reference's solvers are re-entrant: numba
    ``nogil`` kernels on caller-owned arrays).  ``cached`` False: the caller
    closes the private solver when done."""
    dA = as_device_csr(A)
    d = device_inv_diag(pc)
    key = (options.key(), d.data_ptr())
    with _CACHE_LOCK:
        cache = dA.__dict__.setdefault("_solvers", {})
        s = cache.get(key)
        if s is not None and s.lock.acquire(blocking=False):
            return s, True
        if s is None and not any(v.lock.locked() for v in cache.values()):
            s = PipecgSolver(dA, d, options)
            cache.clear()  # one resident solver per matrix bounds HBM use
            cache[key] = s
            s.lock.acquire()
            return s, True
    s = PipecgSolver(dA, d, options)  # busy: a private solver for this call
    s.lock.acquire()
    return s, False


def pipecg_scalars(gamma: float, gamma_prev: float, delta: float, alpha_prev: float,
                   iteration: int) -> tuple[float, float]:
    """Step scalars (alpha, beta) of the pipelined recurrence (solvers.py:276-294).

    The device prologue (csrc/solver.cu ``prologue``) evaluates the same
    expressions in the same order; this host form serves the operator API."""
    if iteration == 0:
        beta = 0.0
        denom = delta
    else:
        beta = gamma / gamma_prev
        denom = delta - beta * gamma / alpha_prev
    if denom == 0.0 or not math.isfinite(denom):
        raise SolverBreakdown("alpha denominator", iteration, denom)
    return gamma / denom, beta


def pipecg_init(A, b, x0, pc) -> PipecgState:
    """Build the pipelined iteration state (solvers.py:297-321) on the device.

    Returns host ndarrays when b is a host array, CUDA tensors otherwise."""
    _check_system(A, b, x0)
    on_dev = is_device_tensor(b)
    x0d = to_device_f64(x0)
    x = x0d.clone()
    r = residual(A, x, to_device_f64(b))
    u = jacobi_apply(pc, r)
    w = spmv(A, u)
    m = jacobi_apply(pc, w)
    n = spmv(A, m)
    gamma, delta, uu = dots([(r, u), (w, u), (u, u)], mode="seq")
    norm = math.sqrt(uu)
    zero = torch.zeros_like(x)
    vecs = dict(x=x, r=r, u=u, w=w, m=m, n=n, z=zero.clone(), q=zero.clone(), s=zero.clone(),
                p=zero.clone())
    if not on_dev:
        vecs = {k: v.cpu().numpy() for k, v in vecs.items()}
    return PipecgState(**vecs, gamma=gamma, gamma_prev=0.0, delta=delta, alpha=0.0,
                       alpha_prev=0.0, beta=0.0, norm=norm)


def pipecg_solve(A, b, x0, pc, cfg: SolverConfig | None = None, *,
                 options: DeviceOptions | None = None, devices=None):
    """Solve Ax = b by pipelined preconditioned CG on the GPU (solvers.py:324-387).

    Same contract and stopping rule as the reference: convergence when
    sqrt((u,u)) < cfg.tolerance, checked at the top of every iteration;
    ``history`` has iterations+1 entries; drift samples every k iterations;
    :class:`SolverBreakdown` on a broken recurrence.  Returns ``(x,
    report)``; x is a host ndarray for host inputs, a CUDA tensor for CUDA
    inputs.

    devices: None (the current GPU) or a list of CUDA device ids; with more
    than one the rows are sharded over them from this process (the
    reference's ``devices=`` keyword, hybrid.py:78; see
    ``distributed.pipecg_solve_devices``)."""
    cfg = cfg or SolverConfig()
    options = options or DeviceOptions()
    t_start = time.perf_counter()
    _check_system(A, b, x0)
    if devices is not None and len(devices) > 1:
        from .distributed import pipecg_solve_devices

        return pipecg_solve_devices(A, b, x0, pc, cfg, devices, options)
    if devices is not None and len(devices) == 1:
        with torch.cuda.device(int(devices[0])):
            return pipecg_solve(A, b, x0, pc, cfg, options=options)
    n = int(A.n_rows)
    on_dev = is_device_tensor(b)
    if n == 0:
        x = torch.zeros(0, dtype=torch.float64, device="cuda") if on_dev else np.zeros(0)
        return x, SolveReport(converged=0.0 < cfg.tolerance, iterations=0, final_norm=0.0,
                              strategy="pipecg", history=[0.0] if cfg.record_history else None,
                              phase_times={"setup": 0.0, "iterations": 0.0},
                              drift_history=[] if cfg.drift_check_interval > 0 else None)
    require_cuda()
    nvtx = torch.cuda.nvtx  # ranges for nsys / Nsight timelines (no-ops otherwise)
    nvtx.range_push("pipecg.setup")
    solver, cached = _solver_for(A, pc, options)
    try:
        bd, x0d = to_device_f64(b), to_device_f64(x0)
        solver.init(bd, x0d, cfg.tolerance, cfg.max_iterations, cfg.drift_check_interval)
        # the solver's stream only: a device-wide synchronize would break a CUDA
        # graph capture of a solver driven from another thread on this GPU
        torch.cuda.ExternalStream(solver.stream).synchronize()
        nvtx.range_pop()
        t_setup = time.perf_counter()
        nvtx.range_push("pipecg.iterations")
        x_out = None if on_dev else _PrefaultedHost(n)  # pages touched while the GPU solves
        res, hist, d_it, d_val = solver.run(cfg.record_history, cfg.max_iterations,
                                            cfg.drift_check_interval)
        nvtx.range_pop()
        t_end = time.perf_counter()
        if res.status == _lib.PCG_BREAKDOWN:
            raise SolverBreakdown(_lib.BREAKDOWN_QUANTITY[res.breakdown_quantity],
                                  int(res.breakdown_iteration), float(res.breakdown_value))
        history = hist[: res.n_history].tolist() if hist is not None else None
        drift = None
        if cfg.drift_check_interval > 0:
            drift = [[int(d_it[k]), float(d_val[k])] for k in range(res.n_drift)]
        x = solver.x_tensor() if on_dev else solver.x_host(out=x_out.get())
    finally:
        solver.lock.release()
        if not cached:
            solver.close()
    report = SolveReport(
        converged=bool(res.converged),
        iterations=int(res.iterations),
        final_norm=float(res.final_norm),
        strategy="pipecg",
        history=history,
        phase_times={"setup": t_setup - t_start, "iterations": t_end - t_setup},
        drift_history=drift,
    )
    return x, report


def true_residual_norm(A, x, b) -> float:
    """Euclidean norm of b - Ax, recomputed from scratch (solvers.py:182-187)."""
    if vec_len(b) != int(A.n_rows):
        raise ValueError("b must have length n_rows")
    return norm2(residual(A, x, b))


def pcg_solve(A, b, x0, pc, cfg: SolverConfig | None = None, *,
              options: DeviceOptions | None = None):
    """Classic PCG (solvers.py:195-273) on the device.

    The reference's baseline algorithm, run like
    :func:`pipecg_solve`: the whole loop on the GPU (csrc/solver.cu engine 4:
    two kernels per iteration -- p update + SpMV + (s, p), then x / r / u
    updates + (u, r), (u, u) -- on-device stop test and breakdown checks,
    CUDA-graph chunks, no per-iteration host synchronisation).  Same
    contract: convergence when sqrt((u, u)) < cfg.tolerance at the top of an
    iteration, ``history`` of iterations + 1 norms, drift every k
    iterations, :class:`SolverBreakdown` ("delta" / "gamma").
    ``options.dot_mode``: "tree" (default) or "seq" (the reference's order:
    bitwise-identical history and x)."""
    cfg = cfg or SolverConfig()
    mode = (options or DeviceOptions()).dot_mode
    t_start = time.perf_counter()
    _check_system(A, b, x0)
    n = int(A.n_rows)
    on_dev = is_device_tensor(b)
    if n == 0:
        x = torch.zeros(0, dtype=torch.float64, device="cuda") if on_dev else np.zeros(0)
        return x, SolveReport(converged=0.0 < cfg.tolerance, iterations=0, final_norm=0.0,
                              strategy="pcg", history=[0.0] if cfg.record_history else None,
                              phase_times={"setup": 0.0, "iterations": 0.0},
                              drift_history=[] if cfg.drift_check_interval > 0 else None)
    require_cuda()
    solver, cached = _solver_for(A, pc, DeviceOptions(dot_mode=mode, engine="pcg"))
    try:
        bd, x0d = to_device_f64(b), to_device_f64(x0)
        solver.init(bd, x0d, cfg.tolerance, cfg.max_iterations, cfg.drift_check_interval)
        torch.cuda.ExternalStream(solver.stream).synchronize()
        t_setup = time.perf_counter()
        x_out = None if on_dev else _PrefaultedHost(n)
        res, hist, d_it, d_val = solver.run(cfg.record_history, cfg.max_iterations,
                                            cfg.drift_check_interval)
        t_end = time.perf_counter()
        if res.status == _lib.PCG_BREAKDOWN:
            raise SolverBreakdown(_lib.BREAKDOWN_QUANTITY[res.breakdown_quantity],
                                  int(res.breakdown_iteration), float(res.breakdown_value))
        history = hist[: res.n_history].tolist() if hist is not None else None
        drift = None
        if cfg.drift_check_interval > 0:
            drift = [[int(d_it[k]), float(d_val[k])] for k in range(res.n_drift)]
        x = solver.x_tensor() if on_dev else solver.x_host(out=x_out.get())
    finally:
        solver.lock.release()
        if not cached:
            solver.close()
    report = SolveReport(
        converged=bool(res.converged), iterations=int(res.iterations),
        final_norm=float(res.final_norm), strategy="pcg", history=history,
        phase_times={"setup": t_setup - t_start, "iterations": t_end - t_setup},
        drift_history=drift,
    )
    return x, report

