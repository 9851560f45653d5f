"""Single-GPU virtual-rank diagnostics for the distributed protocol."""
import sys, threading, time
sys.path.insert(0, '.')
import torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200 import distributed as D

def run(world, kind, n, maxit=300, **opt):
    G = D.LocalGroup(world)
    out, errs = [None]*world, []
    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            prob = D.shard_stencil(kind, n, g)
            xt, b = D.manufactured_local(prob)
            cfg = pb.SolverConfig(tolerance=1e-9, max_iterations=maxit, record_history=True)
            x, rep = D.pipecg_solve_distributed(prob, b, torch.zeros_like(b), cfg, g,
                                                pb.DeviceOptions(**opt))
            out[r] = (rep.iterations, rep.converged, float((x - xt).abs().max()), prob.plan.summary())
        except BaseException as e:
            errs.append((r, repr(e)[:300]))
            G._barrier.abort()
    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    t0 = time.time()
    [t.start() for t in ts]; [t.join(timeout=120) for t in ts]
    print(world, kind, n, opt, 'time %.1fs' % (time.time()-t0), out, errs, flush=True)

if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    if mode == "san":
        run(3, '3d7', 12, maxit=3, use_graphs=False, chunk=1, max_sms=30)
    else:
        for w, n in [(3, 12), (3, 33), (2, 33), (4, 20)]:
            run(w, '3d7', n, use_graphs=False, chunk=1, max_sms=148 // w - 10)
            run(w, '3d7', n, max_sms=148 // w - 10)
