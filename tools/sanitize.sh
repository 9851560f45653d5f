#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck) on small solves of every
# engine: the TMA/mbarrier rings, named barriers and last-block reductions.
OUT=gpurun_out; mkdir -p $OUT
make -s -C paper_2105_06176_b200/csrc >/dev/null 2>&1
cat > /tmp/san_case.py <<'PY'
import sys, math
sys.path.insert(0, ".")
import numpy as np, paper_2105_06176_b200 as pb
eng = sys.argv[1]
def solve(A, b, cfg):
    if eng == "pcg":  # the device PCG (engine 4)
        return pb.pcg_solve(A, b, np.zeros(A.n_rows), pb.jacobi_setup(A), cfg,
                            options=pb.DeviceOptions(chunk=8))
    return pb.pipecg_solve(A, b, np.zeros(A.n_rows), pb.jacobi_setup(A), cfg,
                           options=pb.DeviceOptions(engine=eng, chunk=8))
for kind, n in (("3d7", 20), ("2d5", 64)):
    A = pb.stencil_host(kind, n)
    xt = np.full(A.n_rows, 1 / math.sqrt(A.n_rows)); b = pb.spmv(A, xt)
    x, rep = solve(A, b, pb.SolverConfig(tolerance=1e-9, max_iterations=400))
    print(eng, kind, n, rep.iterations, float(np.abs(x - xt).max()))
P = pb.generate_powerlaw(2**13)
xt = np.full(P.n_rows, 1 / math.sqrt(P.n_rows)); b = pb.spmv(P, xt)
if eng in ("fused-e", "fused-f"):  # diagonal varies by row class: E's code windows
    A = pb.stencil_host("3d7", 14)
    va = np.array(A.values); ro = np.asarray(A.row_offsets); ci = np.asarray(A.col_indices)
    for i in (3, 100, 2000):
        for k in range(ro[i], ro[i + 1]):
            if ci[k] == i: va[k] += 0.5
    A = pb.CsrMatrix(A.n_rows, A.n_cols, ro, ci, va)
    xt = np.full(A.n_rows, 1 / math.sqrt(A.n_rows)); b = pb.spmv(A, xt)
    x, rep = pb.pipecg_solve(A, b, np.zeros(A.n_rows), pb.jacobi_setup(A),
                             pb.SolverConfig(tolerance=1e-9, max_iterations=400),
                             options=pb.DeviceOptions(engine=eng, chunk=8))
    print(eng, "perturbed 3d7", rep.iterations, float(np.abs(x - xt).max()))
    # 125-point: 6,859-entry dictionary, 25 lines bridged into 5 plane windows
    A = pb.stencil_host("p125", 24)
    xt = np.full(A.n_rows, 1 / math.sqrt(A.n_rows)); b = pb.spmv(A, xt)
    x, rep = solve(A, b, pb.SolverConfig(tolerance=1e-9, max_iterations=400))
    print(eng, "p125 24", rep.iterations, float(np.abs(x - xt).max()))
if eng in ("fused-d", "two", "fused-g", "pcg"):  # hub rows: chunks / warp chunks / pcg_hub_kernel
    x, rep = solve(P, b, pb.SolverConfig(tolerance=1e-9, max_iterations=100))
    print(eng, "powerlaw", rep.iterations)
PY
for tool in memcheck racecheck synccheck; do
  for eng in ${ENGINES:-fused-a fused-b fused-c fused-d fused-p fused-e fused-f two fused-g pcg}; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_case.py $eng > $OUT/san_${tool}_${eng}.log 2>&1
    echo "$tool $eng rc=$? $(grep -c 'ERROR SUMMARY: 0 errors\|RACECHECK SUMMARY: 0 hazards' $OUT/san_${tool}_${eng}.log) $(grep 'SUMMARY' $OUT/san_${tool}_${eng}.log | tail -1)"
  done
done
