"""Per-iteration cost of the distributed protocol with ONE rank (no peers):
fused exchange instantiation + last-block publish + arrival spin, vs the
plain single-GPU solver on the same matrix."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200 import distributed as D

kind, n = sys.argv[1], int(sys.argv[2])
g = D.LocalGroup(1).view(0)
for eng in ("fused-a", "fused-c"):
    prob = D.shard_stencil(kind, n, g)
    s = D.DistributedSolver(prob, g, pb.DeviceOptions(engine=eng))
    xt, b = D.manufactured_local(prob)
    s.init(b, torch.zeros_like(b), 0.0, 1000)
    s.solver.enqueue(5); s.solver.prepare(100); torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(s.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.solver.enqueue(100); e1.record(st); e1.synchronize()
    print(kind, n, eng, "distributed(1 rank) ms/iter %.4f" % (e0.elapsed_time(e1) / 100), flush=True)
    s.close()
