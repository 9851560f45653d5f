"""Engine 3 debug: state after k iterations vs engine 2 (seq dots), by row class."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200.solvers import PipecgSolver, DeviceOptions
from paper_2105_06176_b200.kernels import device_inv_diag

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2**12
A = pb.generate_powerlaw(n)
lens = A.row_nnz()
Ad = pb.as_device_csr(A)
pc = pb.jacobi_setup(A)
d = torch.as_tensor(pc.inv_diag, device="cuda")
xt = torch.full((n,), 1 / np.sqrt(n), dtype=torch.float64, device="cuda")
b = pb.spmv(Ad, xt)
out = {}
for eng in ("two", "fused-g"):
    s = PipecgSolver(Ad, d, DeviceOptions(engine=eng, dot_mode="seq"))
    res = {}
    for k in (0, 1, 2, 3):
        s.init(b, torch.zeros_like(b), 0.0, 1000)
        if k:
            s.enqueue(k)
        r = s.poll()
        res[k] = {kk: v.cpu().numpy() for kk, v in s.state_tensors().items()}
        res[k]["_it"] = r.iterations
        res[k]["_eng"] = r.engine
    out[eng] = res
for k in (0, 1, 2, 3):
    a, g = out["two"][k], out["fused-g"][k]
    print("k", k, "engines", a["_eng"], g["_eng"], "its", a["_it"], g["_it"])
    for name in ("x", "r", "u", "w", "z", "q", "s", "p", "m", "n"):
        diff = np.abs(a[name] - g[name])
        bad = np.nonzero(diff > 1e-12 * (np.abs(a[name]).max() + 1e-300))[0]
        cls = lambda idx: (np.sum(lens[idx] > 64), np.sum(lens[idx] <= 64))
        print(f"  {name}: maxdiff {diff.max():.3e} bad {bad.size} (long,short)={cls(bad) if bad.size else ''} first {bad[:8]}")
hub = np.nonzero(lens > 64)[0][:6]
print("hub rows", hub, "lens", lens[hub])
for name in ("x", "u", "p", "z", "n"):
    print(name, "two k1", out["two"][1][name][hub])
    print(name, "G   k1", out["fused-g"][1][name][hub])
print("u k0", out["two"][0]["u"][hub], out["fused-g"][0]["u"][hub])
