"""Row-block sharded PIPECG over several B200s.

The B200 generalisation of the reference's Hybrid-3 split
(/root/reference/pkg/src/pipecg/hybrid.py:418-686, partition.py:55-116):

* P contiguous row blocks balanced by nonzeros -- the P-way form of
  ``decompose_1d`` (partition.py:55-64: cut_p = searchsorted(row_offsets,
  p*nnz/P, 'right') - 1).
* Each rank keeps its rows with columns remapped to a compact local space
  ``[owned rows | halo]`` (halo sorted by global index).  Entry order inside
  a row is untouched -- unlike the reference's local/remote in-row reorder
  (partition.py:67-90), which reassociates row sums (hybrid.py:17-18) -- so
  every row's SpMV stays bitwise equal to the single-device product.
* Per iteration ONE fused kernel (csrc/solver.cu) runs on the local rows
  and does the exchange itself: as each tile's rows are final, its CTA
  stores that tile's halo rows of the vector the peers gather next (w for
  A/E, the stored m for C/D/F) straight into the neighbours' HBM over
  NVLink (CUDA IPC-mapped peer memory); the grid's last block writes the
  rank's dot partial into every rank's slot and bumps every rank's arrival
  counter.  The next iteration's prologue waits for those arrivals -- after
  running the SpMV of a first tile that needs no halo rows, so the
  rendezvous overlaps it (PIPECG's SpMV / reduction overlap).  Only variant
  B keeps a separate exchange kernel.  Drift samples (every k iterations)
  are summed over the ranks in rank order in-kernel.  No host sync, no
  NCCL on the data path; torch.distributed is used only at setup (plan and
  IPC-handle exchange) and to time max-over-ranks.

One process per GPU.  ``LocalGroup`` runs several ranks inside one process
(threads, pointers passed directly) -- the same device protocol, used to
test the exchange on a single GPU.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "nnz_balanced_cuts",
    "HaloPlan",
    "build_plan",
    "remap_columns",
    "ShardedProblem",
    "shard_stencil",
    "shard_csr",
    "shard_block",
    "stencil_block_host",
    "e2e_distributed",
    "DistributedSolver",
    "pipecg_solve_distributed",
    "LocalGroup",
    "TorchGroup",
]


# ---------------------------------------------------------------------------
# partition + halo plan (host logic; unit-tested on CPU with gloo)
# ---------------------------------------------------------------------------
def nnz_balanced_cuts(row_offsets, world: int) -> list[int]:
    """Row cuts [0 = c_0 <= c_1 <= ... <= c_P = N] with prefix nnz(c_p) <=
    p*nnz/P: decompose_1d (partition.py:55-64) applied at every p/P."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    n, nnz = ro.size - 1, int(ro[-1])
    cuts = [0]
    for p in range(1, world):
        target = (nnz * p) // world
        cuts.append(int(np.searchsorted(ro, target, side="right") - 1))
    cuts.append(n)
    for p in range(1, world + 1):  # keep monotone (degenerate rows)
        cuts[p] = max(cuts[p], cuts[p - 1])
    return cuts


def stencil_cuts(prefix, n_rows: int, world: int) -> list[int]:
    """nnz-balanced cuts from a closed-form prefix count (no host CSR)."""
    nnz = prefix(n_rows)
    cuts = [0]
    for p in range(1, world):
        target = (nnz * p) // world
        lo, hi = cuts[-1], n_rows  # largest k with prefix(k) <= target
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if prefix(mid) <= target:
                lo = mid
            else:
                hi = mid - 1
        cuts.append(lo)
    cuts.append(n_rows)
    return cuts


def owner_of(cols: np.ndarray, cuts: list[int]) -> np.ndarray:
    return np.searchsorted(np.asarray(cuts[1:], dtype=np.int64), cols, side="right")


@dataclass
class HaloPlan:
    rank: int
    world: int
    cuts: list
    n_local: int
    halo_cols: np.ndarray          # sorted global columns this rank reads but does not own
    send_row: np.ndarray           # local rows this rank sends ...
    send_peer: np.ndarray          # ... to these ranks ...
    send_dst: np.ndarray           # ... at these indices of the peer's local column space

    @property
    def row_begin(self) -> int:
        return int(self.cuts[self.rank])

    @property
    def row_end(self) -> int:
        return int(self.cuts[self.rank + 1])

    @property
    def n_halo(self) -> int:
        return int(self.halo_cols.size)

    @property
    def n_cols_local(self) -> int:
        return self.n_local + self.n_halo

    def summary(self) -> dict:
        return {"rank": self.rank, "world": self.world, "rows": [self.row_begin, self.row_end],
                "n_halo": self.n_halo, "n_send": int(self.send_row.size),
                "halo_bytes_per_iteration": 8 * int(self.send_row.size)}


def remap_columns(cols_global, row_begin: int, row_end: int):
    """Global columns -> local [owned | halo] indices; returns (local, halo).

    Works on numpy arrays or CUDA torch tensors (setup-time index work)."""
    n_local = row_end - row_begin
    try:
        import torch

        if isinstance(cols_global, torch.Tensor):
            c = cols_global.to(torch.int64)
            outside = (c < row_begin) | (c >= row_end)
            halo = torch.unique(c[outside])
            pos = torch.searchsorted(halo, c)
            local = torch.where(outside, n_local + pos, c - row_begin)
            return local.to(torch.int32), halo.cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    c = np.asarray(cols_global, dtype=np.int64)
    outside = (c < row_begin) | (c >= row_end)
    halo = np.unique(c[outside])
    local = np.where(outside, n_local + np.searchsorted(halo, c), c - row_begin)
    return local.astype(np.int64), halo


def build_plan(rank: int, world: int, cuts: list[int], halo_cols: np.ndarray, group) -> HaloPlan:
    """Each rank announces the halo columns it needs (grouped by owner) and
    where it stores them; each rank then derives what it must send."""
    n_local = int(cuts[rank + 1] - cuts[rank])
    halo_cols = np.asarray(halo_cols, dtype=np.int64)
    owners = owner_of(halo_cols, cuts)
    requests = {}
    for q in np.unique(owners):
        sel = np.nonzero(owners == q)[0]
        requests[int(q)] = (halo_cols[sel], n_local + sel.astype(np.int64))
    all_requests = group.all_gather_object(requests)
    rows, peers, dsts = [], [], []
    for q, req in enumerate(all_requests):
        if rank in req:
            cols, dst = req[rank]
            rows.append(np.asarray(cols, dtype=np.int64) - cuts[rank])
            peers.append(np.full(len(cols), q, dtype=np.int64))
            dsts.append(np.asarray(dst, dtype=np.int64))
    cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, dtype=np.int64))
    send_row, send_peer, send_dst = cat(rows), cat(peers), cat(dsts)
    if send_row.size and (send_row.min() < 0 or send_row.max() >= n_local):
        raise ValueError("a peer requested a row this rank does not own")
    return HaloPlan(rank, world, list(cuts), n_local, halo_cols, send_row, send_peer, send_dst)


def exchange_values(plan: HaloPlan, local_values: np.ndarray, group) -> np.ndarray:
    """Host-side halo exchange (setup only, e.g. inv_diag): returns the halo
    values in this rank's halo order."""
    out_msgs = {}
    for q in np.unique(plan.send_peer):
        sel = plan.send_peer == q
        out_msgs[int(q)] = (plan.send_dst[sel], local_values[plan.send_row[sel]])
    msgs = group.all_gather_object(out_msgs)
    halo = np.zeros(plan.n_halo)
    for q, m in enumerate(msgs):
        if plan.rank in m:
            dst, vals = m[plan.rank]
            halo[np.asarray(dst) - plan.n_local] = vals
    return halo


# ---------------------------------------------------------------------------
# process groups
# ---------------------------------------------------------------------------
class TorchGroup:
    """torch.distributed (nccl or gloo) as the setup-time object transport."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.local = False

    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)

    def max(self, value: float) -> float:
        import torch

        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


class LocalGroup:
    """Several ranks in ONE process (one thread per rank); all_gather_object
    is a rendezvous between the threads.  Device pointers are exchanged
    directly instead of through CUDA IPC."""

    def __init__(self, world: int):
        self.world = world
        self._barrier = threading.Barrier(world)
        self._slots = [None] * world
        self.local = True

    def view(self, rank: int) -> "_LocalRank":
        return _LocalRank(self, rank)


class _LocalRank:
    def __init__(self, parent: LocalGroup, rank: int):
        self.parent, self.rank, self.world, self.local = parent, rank, parent.world, True

    def all_gather_object(self, obj):
        p = self.parent
        p._slots[self.rank] = obj
        p._barrier.wait()
        out = list(p._slots)
        p._barrier.wait()
        return out

    def barrier(self):
        self.parent._barrier.wait()

    def max(self, value: float) -> float:
        return max(self.all_gather_object(value))


# ---------------------------------------------------------------------------
# sharded problems
# ---------------------------------------------------------------------------
@dataclass
class ShardedProblem:
    """One rank's share: local CSR (local column indices), plan, inv_diag
    over [owned | halo], and the global sizes."""

    plan: HaloPlan
    A: object                 # DeviceCsr with n_cols = n_local + n_halo
    inv_diag: object          # CUDA float64 tensor, n_local + n_halo
    global_rows: int
    global_nnz: int
    meta: dict = field(default_factory=dict)


def _localize(dA, row_begin: int, row_end: int):
    import torch

    local, halo = remap_columns(dA.col[: dA.nnz], row_begin, row_end)
    dA.col[: dA.nnz].copy_(local)
    dA.n_cols = (row_end - row_begin) + halo.size
    del local
    torch.cuda.empty_cache()
    return halo


def _finish(dA, plan: HaloPlan, group, global_rows, global_nnz, meta=None) -> ShardedProblem:
    import torch

    from .kernels import jacobi_setup

    # inv_diag of owned rows: the diagonal sits at local column == local row
    sq = type(dA)(dA.n_rows, dA.n_rows, dA.nnz, dA.rowptr, dA.col, dA.val)
    d_local = jacobi_setup(sq).inv_diag  # CUDA tensor (n_local)
    halo_vals = exchange_values(plan, d_local.cpu().numpy(), group)
    d = torch.empty(plan.n_cols_local, dtype=torch.float64, device=d_local.device)
    d[: plan.n_local].copy_(d_local)
    if plan.n_halo:
        d[plan.n_local:].copy_(torch.from_numpy(halo_vals))
    return ShardedProblem(plan, dA, d, global_rows, global_nnz, meta or {})


def shard_stencil(kind, n: int, group) -> ShardedProblem:
    """Generate this rank's nnz-balanced row block of a stencil in HBM."""
    from . import sparse

    k = sparse._KINDS[kind]
    N, nnz = sparse.stencil_shape(k, n)
    cuts = stencil_cuts(lambda r: sparse._prefix_count(k, n, r), N, group.world)
    r0, r1 = cuts[group.rank], cuts[group.rank + 1]
    dA = sparse.stencil_device(k, n, r0, r1)
    halo = _localize(dA, r0, r1)
    plan = build_plan(group.rank, group.world, cuts, halo, group)
    return _finish(dA, plan, group, N, nnz, {"kind": kind, "n": n})


def shard_csr(A, group) -> ShardedProblem:
    """This rank's nnz-balanced row block of a host CSR matrix (duck-typed
    CsrMatrix), uploaded and localized."""
    ro = np.asarray(A.row_offsets, dtype=np.int64)
    cuts = nnz_balanced_cuts(ro, group.world)
    r0, r1 = cuts[group.rank], cuts[group.rank + 1]
    lo, hi = int(ro[r0]), int(ro[r1])

    class _Block:
        n_rows = r1 - r0
        n_cols = int(A.n_cols)
        row_offsets = ro[r0: r1 + 1] - lo
        col_indices = np.asarray(A.col_indices)[lo:hi]
        values = np.asarray(A.values)[lo:hi]

    return shard_block(_Block, cuts, group, int(A.n_rows), int(ro[-1]))


def shard_block(block, cuts, group, global_rows: int, global_nnz: int, meta=None) -> ShardedProblem:
    """This rank's rows [cuts[rank], cuts[rank+1]) given as host CSR arrays
    with GLOBAL column indices (the caller's own block: nothing global is
    materialised anywhere), uploaded through the pinned pipeline and
    localized to [owned | halo]."""
    from .sparse import DeviceCsr, upload_csr

    r0, r1 = cuts[group.rank], cuts[group.rank + 1]
    dA = upload_csr(block)
    assert isinstance(dA, DeviceCsr)
    halo = _localize(dA, r0, r1)
    plan = build_plan(group.rank, group.world, cuts, halo, group)
    return _finish(dA, plan, group, global_rows, global_nnz, meta)


def stencil_block_host(kind, n: int, group):
    """(block, cuts, N, nnz): this rank's stencil row block as host arrays
    with global columns -- the input of the host-buffer (e2e) path."""
    from . import sparse

    k = sparse._KINDS[kind]
    N, nnz = sparse.stencil_shape(k, n)
    cuts = stencil_cuts(lambda r: sparse._prefix_count(k, n, r), N, group.world)
    r0, r1 = cuts[group.rank], cuts[group.rank + 1]
    d = sparse.stencil_device(k, n, r0, r1)
    block = d.to_host()
    del d
    return block, cuts, N, nnz


def e2e_distributed(kind, n: int, group, tolerance: float, max_iterations: int = 20000,
                    block=None, options=None):
    """The multi-GPU public call with host buffers: this rank's host block
    -> upload + localize + halo plan + connect + solve + x download.
    Returns (iterations, seconds (max over ranks), h2d bytes of this rank,
    d2h bytes of this rank, max |x - x_true| over ranks)."""
    import torch

    from .solvers import SolverConfig

    from ._device import d2h, to_device_f64

    block, cuts, N, nnz = block or stencil_block_host(kind, n, group)
    r0, r1 = cuts[group.rank], cuts[group.rank + 1]
    x_true = np.full(r1 - r0, 1.0 / math.sqrt(N))
    # the caller's right-hand side b = A x_true as a host array (not timed)
    prob0 = shard_block(block, cuts, group, N, nnz)
    b_host = d2h(manufactured_local(prob0)[1])
    del prob0
    torch.cuda.empty_cache()
    x0_host = np.zeros(r1 - r0)
    group.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = shard_block(block, cuts, group, N, nnz)
    b = to_device_f64(b_host)
    x, rep = pipecg_solve_distributed(prob, b, to_device_f64(x0_host),
                                      SolverConfig(tolerance=tolerance,
                                                   max_iterations=max_iterations), group,
                                      options=options)
    x_host = d2h(x)
    dt = time.perf_counter() - t0
    err = float(np.max(np.abs(x_host - x_true))) if x_host.size else 0.0
    rp = 8 if block.nnz >= 2**31 else 4
    h2d = rp * (block.n_rows + 1) + 12 * block.nnz + 16 * (r1 - r0)
    return rep.iterations, group.max(dt), h2d, 8 * x_host.size, group.max(err)


# ---------------------------------------------------------------------------
# the distributed solver
# ---------------------------------------------------------------------------
class DistributedSolver:
    """Native solver on this rank's block, connected to its peers."""

    def __init__(self, problem: ShardedProblem, group, options=None):
        import torch

        from . import _lib
        from .solvers import DeviceOptions, PipecgSolver

        self.problem, self.group = problem, group
        opts = options or DeviceOptions()
        if opts.engine in ("two", "fused-g"):
            raise ValueError("the distributed path runs the fused engine (variants A-F)")
        engine = opts.engine if opts.engine.startswith("fused") else "fused"
        opts = DeviceOptions(dot_mode=opts.dot_mode, engine=engine, chunk=opts.chunk,
                             use_graphs=opts.use_graphs, max_sms=opts.max_sms)
        try:
            self.solver = PipecgSolver(problem.A, problem.inv_diag, opts)
        except _lib.NativeError:
            # E/F asked for, but this shard has no row-pattern dictionary
            if engine not in ("fused-e", "fused-f"):
                raise
            opts.engine = "fused-a" if engine == "fused-e" else "fused-c"
            self.solver = PipecgSolver(problem.A, problem.inv_diag, opts)
        # every rank must run the same fused variant: the exchange pushes the
        # vector the variant gathers (w for A/B, the stored m for C/D), and
        # per-rank autotuning could pick differently on differently shaped
        # blocks -> adopt rank 0's choice
        # (E/F keep their row-pattern windows across the shard's halo; a rank
        # that cannot run rank 0's E/F runs the CSR variant that pushes the
        # same vector: E -> A (w), F -> C (m))
        names = {3: "fused-a", 4: "fused-b", 5: "fused-c", 6: "fused-d", 8: "fused-e",
                 9: "fused-f"}
        mine = int(self.solver.poll().engine)
        mine = 5 if mine == 7 else mine  # P runs as C once connected
        chosen = group.all_gather_object(mine)[0]
        # Connected, E (staged layout, csrc/solver.cu solver_connect) beats F
        # wherever measured (tools/dist1.py, one B200): 3D 7-pt 256^3 one
        # rank E 0.339 / F 0.412 ms per iteration, two virtual ranks 0.389 /
        # 1.242, 27-pt 300^3 one rank 0.694 / 1.290 -- F's consumer-loaded
        # streams do not mix with the fused exchange.  So an autotuned F
        # (rank 0's single-GPU pick) runs as E once connected.
        if (chosen == 9 and engine != "fused-f"
                and not os.environ.get("PIPECG_B200_DIST_KEEP_F")):
            chosen = 8
        if mine != chosen:
            self.solver.close()
            opts = DeviceOptions(dot_mode=opts.dot_mode, engine=names[chosen], chunk=opts.chunk,
                                 use_graphs=opts.use_graphs, max_sms=opts.max_sms)
            try:
                self.solver = PipecgSolver(problem.A, problem.inv_diag, opts)
            except _lib.NativeError:
                if chosen not in (8, 9):
                    raise
                opts.engine = names[3 if chosen == 8 else 5]
                self.solver = PipecgSolver(problem.A, problem.inv_diag, opts)
        vbuf, ld, comm = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_void_p()
        _lib.call("pipecg_b200_solver_comm_info", self.solver._h, ctypes.byref(vbuf),
                  ctypes.byref(ld), ctypes.byref(comm))
        self._opened = []
        if getattr(group, "local", False):
            infos = group.all_gather_object((vbuf.value, ld.value, comm.value))
            peer_vbuf = [i[0] for i in infos]
            peer_comm = [i[2] for i in infos]
        else:
            hv, hc = (ctypes.c_char * 64)(), (ctypes.c_char * 64)()
            _lib.call("pipecg_b200_ipc_get_handle", vbuf, hv)
            _lib.call("pipecg_b200_ipc_get_handle", comm, hc)
            infos = group.all_gather_object((bytes(hv), ld.value, bytes(hc)))
            peer_vbuf, peer_comm = [], []
            for q, (hvq, _, hcq) in enumerate(infos):
                if q == group.rank:
                    peer_vbuf.append(vbuf.value)
                    peer_comm.append(comm.value)
                    continue
                pv, pc = ctypes.c_void_p(), ctypes.c_void_p()
                _lib.call("pipecg_b200_ipc_open", ctypes.create_string_buffer(hvq, 64),
                          ctypes.byref(pv))
                _lib.call("pipecg_b200_ipc_open", ctypes.create_string_buffer(hcq, 64),
                          ctypes.byref(pc))
                self._opened += [pv.value, pc.value]
                peer_vbuf.append(pv.value)
                peer_comm.append(pc.value)
        W = group.world
        # (kept for diagnostics: the addresses this rank pushes to)
        self.comm_ptr, self.peer_comm, self.peer_vbuf = comm.value, list(peer_comm), list(peer_vbuf)
        plan = problem.plan
        dev = problem.inv_diag.device
        self._send = [torch.from_numpy(plan.send_row.astype(np.int32)).to(dev),
                      torch.from_numpy(plan.send_peer.astype(np.int32)).to(dev),
                      torch.from_numpy(plan.send_dst.astype(np.int64)).to(dev)]
        _lib.call("pipecg_b200_solver_connect", self.solver._h, group.rank, W,
                  (ctypes.c_void_p * W)(*peer_vbuf), (ctypes.c_int64 * W)(*[i[1] for i in infos]),
                  (ctypes.c_void_p * W)(*peer_comm), int(plan.send_row.size),
                  self._send[0].data_ptr(), self._send[1].data_ptr(), self._send[2].data_ptr())
        group.barrier()

    def close(self):
        from . import _lib

        L = _lib.load()
        for p in self._opened:
            L.pipecg_b200_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        self.solver.close()

    def init(self, b_local, x0_local, tolerance: float, max_iterations: int,
             drift_check_interval: int = 0):
        import torch

        # every rank's previous GPU work (including exchanges still landing
        # in peers' memory) has drained before anyone re-arms its counters
        torch.cuda.current_stream().synchronize()
        self.solver.poll()
        self.group.barrier()
        self.solver.init(b_local, x0_local, tolerance, max_iterations, drift_check_interval)

    def run(self, record_history: bool, max_iterations: int, drift_check_interval: int = 0):
        """Drift samples (drift_check_interval > 0): every rank's rows, summed
        over the ranks in rank order in-kernel (csrc/solver.cu
        drift_push_kernel / drift_dist_finish_kernel): the same values on
        every rank, solvers.py:190-192,371-372."""
        return self.solver.run(record_history, max_iterations, drift_check_interval)

    @property
    def stream(self) -> int:
        return self.solver.stream

    def x_local(self):
        return self.solver.x_tensor()


def manufactured_local(problem: ShardedProblem):
    """x_true = 1/sqrt(N) on the owned rows and b = A x_true (cli.py:83-100);
    x_true is constant, so the halo of x_true is the same constant."""
    import torch

    from .kernels import spmv

    n_glob = problem.global_rows
    xt = torch.full((problem.plan.n_cols_local,), 1.0 / math.sqrt(n_glob), dtype=torch.float64,
                    device=problem.inv_diag.device)
    b = spmv(problem.A, xt)
    return xt[: problem.plan.n_local].clone(), b


def pipecg_solve_distributed(problem: ShardedProblem, b_local, x0_local, cfg, group,
                             options=None, solver: DistributedSolver | None = None):
    """pipecg_solve on a row-sharded problem; every rank returns its local
    block of x and the same SolveReport (solvers.py:324-387 semantics)."""
    from . import _lib
    from .solvers import SolveReport, SolverBreakdown, SolverConfig

    cfg = cfg or SolverConfig()
    own = solver is None
    solver = solver or DistributedSolver(problem, group, options)
    t0 = time.perf_counter()
    solver.init(b_local, x0_local, cfg.tolerance, cfg.max_iterations, cfg.drift_check_interval)
    import torch

    # the solver's own stream, not the device: another rank sharing this GPU
    # (devices=[0, 0], virtual ranks) may be capturing a CUDA graph, and a
    # device-wide synchronize would invalidate that capture
    torch.cuda.ExternalStream(solver.stream).synchronize()
    t1 = time.perf_counter()
    res, hist, d_it, d_val = solver.run(cfg.record_history, cfg.max_iterations,
                                        cfg.drift_check_interval)
    t2 = time.perf_counter()
    x = solver.x_local()
    if own:
        solver.close()
    if res.status == _lib.PCG_BREAKDOWN:
        raise SolverBreakdown(_lib.BREAKDOWN_QUANTITY[res.breakdown_quantity],
                              int(res.breakdown_iteration), float(res.breakdown_value))
    rep = SolveReport(
        converged=bool(res.converged), iterations=int(res.iterations),
        final_norm=float(res.final_norm), strategy="pipecg",
        history=hist[: res.n_history].tolist() if hist is not None else None,
        phase_times={"setup": t1 - t0, "iterations": t2 - t1},
        drift_history=([[int(d_it[k]), float(d_val[k])] for k in range(res.n_drift)]
                       if cfg.drift_check_interval > 0 else None),
        partition=problem.plan.summary(),
    )
    return x, rep


def pipecg_solve_devices(A, b, x0, pc, cfg, devices, options=None):
    """``pipecg_solve(..., devices=[d0, d1, ...])`` from ONE process (the
    reference's ``devices=`` keyword, hybrid.py:78,235,424):
    one thread per device, the host CSR split into nnz-balanced row blocks
    (``shard_csr``), peer access enabled between the devices, and the same
    fused exchange as the one-process-per-GPU path -- every device pushes its
    halo rows and dot partials straight into the others' memory.  Returns the
    gathered x (host ndarray, or a CUDA tensor on devices[0] for CUDA inputs)
    and rank 0's SolveReport (identical on every rank).  A device listed
    twice shares that GPU (grids sized for co-residency; used by the tests)."""
    import torch

    from . import _lib
    from .solvers import DeviceOptions, SolverBreakdown, SolverConfig, is_device_tensor

    cfg = cfg or SolverConfig()
    devices = [int(d) for d in devices]
    W = len(devices)
    on_dev = is_device_tensor(b)
    host = A.to_host() if hasattr(A, "to_host") else A
    bh = b.detach().cpu().numpy() if on_dev else np.ascontiguousarray(b, dtype=np.float64)
    xh = (x0.detach().cpu().numpy() if is_device_tensor(x0)
          else np.ascontiguousarray(x0, dtype=np.float64))
    d = pc.inv_diag
    dh = d.detach().cpu().numpy() if is_device_tensor(d) else np.asarray(d, dtype=np.float64)
    opts = options or DeviceOptions()
    if len(set(devices)) < W:  # a GPU shared by several ranks: co-resident grids
        from ._device import shared_max_sms

        share = max(devices.count(dv) for dv in set(devices))
        busiest = max(set(devices), key=devices.count)
        opts = DeviceOptions(dot_mode=opts.dot_mode, engine=opts.engine, chunk=opts.chunk,
                             use_graphs=opts.use_graphs, max_sms=shared_max_sms(share, busiest))
    for dv in set(devices):
        for q in set(devices):
            if q != dv:
                _lib.call("pipecg_b200_enable_peer_access", dv, q)
    G = LocalGroup(W)
    out, errs = [None] * W, []

    def work(r):
        try:
            torch.cuda.set_device(devices[r])
            g = G.view(r)
            prob = shard_csr(host, g)
            r0, r1 = prob.plan.row_begin, prob.plan.row_end
            # the caller's preconditioner on [owned | halo] (not the shard's own Jacobi)
            dl = np.concatenate([dh[r0:r1], dh[prob.plan.halo_cols]])
            prob.inv_diag.copy_(torch.from_numpy(dl))
            dev = prob.inv_diag.device
            bl = torch.from_numpy(bh[r0:r1].copy()).to(dev)
            xl = torch.from_numpy(xh[r0:r1].copy()).to(dev)
            x, rep = pipecg_solve_distributed(prob, bl, xl, cfg, g, opts)
            out[r] = (x.cpu().numpy(), rep)
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        first = sorted(errs, key=lambda e: isinstance(e[1], threading.BrokenBarrierError))[0][1]
        if isinstance(first, SolverBreakdown):
            raise first
        raise RuntimeError(f"pipecg_solve(devices={devices}) failed: {first!r}") from first
    x = np.concatenate([o[0] for o in out])
    rep = out[0][1]
    if on_dev:
        x = torch.from_numpy(x).to(torch.device("cuda", devices[0]))
    return x, rep
