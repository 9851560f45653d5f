"""cProfile of the FIRST pipecg_solve call on a host CSR (autotune + first use)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200._device import warm_transfers

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = pb.stencil_device("3d7", n).to_host()
N = A.n_rows
b = pb.spmv(A, np.full(N, 1.0 / np.sqrt(N)))
pc = pb.jacobi_setup(A)
warm_transfers()
tol = 1e-8 * float(np.linalg.norm(b))
A2 = pb.CsrMatrix(N, N, A.row_offsets.copy(), A.col_indices.copy(), A.values.copy())
P2 = pb.JacobiPreconditioner(pc.inv_diag.copy())
pr = cProfile.Profile()
pr.enable()
t = time.perf_counter()
x, rep = pb.pipecg_solve(A2, b, np.zeros(N), P2, pb.SolverConfig(tolerance=tol, max_iterations=1))
dt = time.perf_counter() - t
pr.disable()
print("first call", dt, rep.phase_times)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
