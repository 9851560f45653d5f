import sys, math
sys.path.insert(0, ".")
import numpy as np, paper_2105_06176_b200 as pb
eng, kind, n, chunk = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
A = pb.stencil_host(kind, n)
xt = np.full(A.n_rows, 1 / math.sqrt(A.n_rows)); b = pb.spmv(A, xt)
x, rep = pb.pipecg_solve(A, b, np.zeros(A.n_rows), pb.jacobi_setup(A),
                         pb.SolverConfig(tolerance=1e-300, max_iterations=6),
                         options=pb.DeviceOptions(engine=eng, chunk=chunk))
print(eng, kind, n, rep.iterations)
