"""First-call cost of pipecg_solve on a host CSR (3D 7-pt 256^3): setup phase
times printed by the library (PIPECG_B200_DEBUG_PLAN=1), then a second call
for comparison."""
import os, sys, time
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
for k in range(2):
    A2 = pb.CsrMatrix(N, N, A.row_offsets.copy(), A.col_indices.copy(), A.values.copy())
    t = time.perf_counter()
    x, rep = pb.pipecg_solve(A2, b, np.zeros(N), pb.JacobiPreconditioner(pc.inv_diag.copy()),
                             pb.SolverConfig(tolerance=1e-8 * float(np.linalg.norm(b))))
    dt = time.perf_counter() - t
    print(f"call {k}: {dt*1e3:.1f} ms, {rep.iterations} it, setup {rep.phase_times['setup']*1e3:.1f} ms", flush=True)
