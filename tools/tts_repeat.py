import sys, math, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2105_06176_b200 as pb
A = pb.stencil_device("3d7", 256)
N = A.n_rows
xt = torch.full((N,), 1 / math.sqrt(N), dtype=torch.float64, device="cuda")
b = pb.spmv(A, xt)
pc = pb.jacobi_setup(A)
u0 = pb.jacobi_apply(pc, b)
tol = 1e-8 * math.sqrt(pb.dot(u0, u0, mode="tree"))
for k in range(4):
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x, rep = pb.pipecg_solve(A, b, torch.zeros_like(b), pc, cfg)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(k, rep.iterations, "setup %.1f ms iters %.1f ms (%.4f ms/it) total %.1f" % (rep.phase_times["setup"]*1e3, rep.phase_times["iterations"]*1e3, rep.phase_times["iterations"]*1e3/rep.iterations, (t1-t0)*1e3), flush=True)
