import sys; sys.path.insert(0,'.')
import numpy as np, paper_2105_06176_b200 as pb
A = pb.stencil_host("3d7", 24)
pc = pb.jacobi_setup(A)
b = np.ones(A.n_rows)
x, rep = pb.pipecg_solve(A, b, np.zeros(A.n_rows), pc, pb.SolverConfig(tolerance=1e-8, max_iterations=50), options=pb.DeviceOptions(engine="fused-e"))
print("ok", rep.iterations)
