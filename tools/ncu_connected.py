"""One connected rank (world 1) at 3D 7-pt 256^3, E in a given layout, 12
iterations -- a target for ncu (PIPECG_B200_DIST_KEEP_DV=1 keeps the
consumer-loaded layout)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200 import distributed as D

G = D.LocalGroup(1)
g = G.view(0)
prob = D.shard_stencil("3d7", 256, g)
s = D.DistributedSolver(prob, g, pb.DeviceOptions(engine="fused-e"))
xt, b = D.manufactured_local(prob)
s.init(b, torch.zeros_like(b), 0.0, 12)
res = s.run(False, 12)[0]
print("flags", res.pattern_flags, "it", res.iterations)
s.close()
