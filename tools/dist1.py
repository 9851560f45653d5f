"""Per-iteration cost of the distributed protocol on ONE GPU.

    python tools/dist1.py 3d7 256 [engines=fused-a,fused-c,fused-e,fused-f] [world=1]

world=1: one rank, no peers (fused exchange instantiation + last-block
publish + arrival spin) vs the plain single-GPU solver on the same matrix.
world>1: that many virtual ranks as threads sharing the GPU (grids sized
for co-residency, so the ranks split the SMs and the HBM bandwidth): the
halo windows / pushes / waits are exercised; ms/iter is the max over ranks.
"""
import sys, threading
sys.path.insert(0, ".")
import torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200._device import shared_max_sms
from paper_2105_06176_b200 import distributed as D

kind, n = sys.argv[1], int(sys.argv[2])
engines = sys.argv[3].split(",") if len(sys.argv) > 3 else ["fused-a", "fused-c", "fused-e", "fused-f"]
world = int(sys.argv[4]) if len(sys.argv) > 4 else 1
for eng in engines:
    G = D.LocalGroup(world)
    opts = pb.DeviceOptions(engine=eng, max_sms=0 if world == 1 else shared_max_sms(world))
    ms, info, errs = [0.0] * world, [None] * world, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            g = G.view(r)
            prob = D.shard_stencil(kind, n, g)
            s = D.DistributedSolver(prob, g, opts)
            xt, b = D.manufactured_local(prob)
            s.init(b, torch.zeros_like(b), 0.0, 1000)
            s.solver.enqueue(5); s.solver.prepare(100)
            torch.cuda.ExternalStream(s.stream).synchronize()  # not the device: peers may capture
            g.barrier()
            st = torch.cuda.ExternalStream(s.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); s.solver.enqueue(100); e1.record(st); e1.synchronize()
            ms[r] = e0.elapsed_time(e1) / 100
            res = s.solver.poll()
            info[r] = (res.engine, res.pattern_flags)
            g.barrier()
            s.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(repr(e))
            G._barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    print(kind, n, eng, f"world={world}", "errors" if errs else f"ms/iter {max(ms):.4f}",
          info, errs[:1], flush=True)
