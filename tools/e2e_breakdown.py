"""Phase timing of the reference-facing call with host buffers (e2e leg)."""
import math, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200 import solvers as S, kernels as K, sparse as SP

kind, n = sys.argv[1], int(sys.argv[2])
Ad = pb.stencil_device(kind, n)
Ah = Ad.to_host()
del Ad
torch.cuda.empty_cache()
N = Ah.n_rows
x_true = np.full(N, 1 / math.sqrt(N))
b = pb.spmv(Ah, x_true)
d = pb.jacobi_setup(Ah).inv_diag
u0 = d * b
tol = 1e-8 * math.sqrt(float(np.dot(u0, u0)))
for rep in range(3):
    A = pb.CsrMatrix.__new__(pb.CsrMatrix)
    for k, v in (("n_rows", N), ("n_cols", N), ("row_offsets", Ah.row_offsets),
                 ("col_indices", Ah.col_indices), ("values", Ah.values)):
        object.__setattr__(A, k, v)
    pc = pb.JacobiPreconditioner(d)
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    dA = SP.as_device_csr(A); torch.cuda.synchronize(); t.append(time.perf_counter())
    dd = K.device_inv_diag(pc); torch.cuda.synchronize(); t.append(time.perf_counter())
    s, _ = S._solver_for(A, pc, pb.DeviceOptions()); s.lock.release(); torch.cuda.synchronize(); t.append(time.perf_counter())
    bd, x0d = pb.solvers.to_device_f64(b), pb.solvers.to_device_f64(np.zeros(N)); torch.cuda.synchronize(); t.append(time.perf_counter())
    s.init(bd, x0d, tol, 20000, 0); torch.cuda.synchronize(); t.append(time.perf_counter())
    res = s.run(False, 20000, 0)[0]; t.append(time.perf_counter())
    x = s.x_host(); t.append(time.perf_counter())
    names = ["upload_csr", "inv_diag", "solver_create(autotune)", "b,x0 upload", "init", "run", "x download"]
    print(kind, n, "iters", res.iterations, " ".join(f"{nm}={1e3*(t[i+1]-t[i]):.1f}ms" for i, nm in enumerate(names)),
          f"total={1e3*(t[-1]-t[0]):.1f}ms", flush=True)
    s.close(); del s, dA, A, pc, dd, bd, x0d
    torch.cuda.empty_cache()
