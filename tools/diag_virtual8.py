"""Reproduce the rare 8-virtual-rank setup stall with diagnostics: every
rank's comm pointer, the peer pointers it pushes to, and every comm
buffer's arrival counters when a solve times out."""
import gc, sys, threading, time
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np, torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200 import distributed as D
from paper_2105_06176_b200._device import shared_max_sms


class _Ptr:
    def __init__(self, p, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u8", "data": (p, False),
                                         "version": 3}


def counters(p):
    return torch.as_tensor(_Ptr(p, 4), device="cuda").cpu().tolist()


# host timestamps around each rank's init phases (monkeypatched)
T = {}
_orig_init = D.DistributedSolver.init


def _timed_init(self, b, x0, tol, maxit, drift=0):
    r = self.group.rank
    torch.cuda.current_stream().synchronize()
    T[(r, "pre_poll")] = time.perf_counter()
    self.solver.poll()
    T[(r, "pre_barrier")] = time.perf_counter()
    self.group.barrier()
    T[(r, "post_barrier")] = time.perf_counter()
    self.solver.init(b, x0, tol, maxit, drift)
    T[(r, "init_returned")] = time.perf_counter()


D.DistributedSolver.init = _timed_init
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = pb.SolverConfig(tolerance=1e-9, max_iterations=3000)
world, kind, n, eng = 8, "3d7", 40, "fused-a"
fails = 0
for rep in range(reps):
    G = D.LocalGroup(world)
    T.clear()
    solvers, errs, engines = [None] * world, [], [None] * world
    opts = pb.DeviceOptions(max_sms=shared_max_sms(world), engine=eng)

    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            prob = D.shard_stencil(kind, n, g)
            xt, b = D.manufactured_local(prob)
            s = D.DistributedSolver(prob, g, opts)
            solvers[r] = s
            engines[r] = int(s.solver.poll().engine)
            D.pipecg_solve_distributed(prob, b, torch.zeros_like(b), cfg, g, solver=s)
        except BaseException as e:  # noqa: BLE001
            errs.append((r, repr(e)[:200]))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if errs:
        t0 = min(v for v in T.values())
        for r in range(world):
            print(f"  rank {r} times: " + " ".join(
                f"{k}={T[(r, k)] - t0:.3f}" for k in ("pre_poll", "pre_barrier", "post_barrier",
                                                       "init_returned") if (r, k) in T), flush=True)
    if errs:
        fails += 1
        print(f"rep {rep}: FAIL engines {engines}", flush=True)
        for r, e in sorted(errs):
            print(f"  rank {r}: {e}", flush=True)
        for r, s in enumerate(solvers):
            if s is None:
                print(f"  rank {r}: no solver"); continue
            own = s.comm_ptr
            bad = [q for q in range(world) if solvers[q] is not None and s.peer_comm[q] != solvers[q].comm_ptr]
            print(f"  rank {r}: comm {own:#x} counters {counters(own)} peers-mismatch {bad}", flush=True)
    for s in solvers:
        if s is not None:
            s.close()
    del solvers
    gc.collect()
print(f"{fails} failures in {reps} solves", flush=True)
