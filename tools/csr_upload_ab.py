"""CSR upload of the 3D 7-pt 256^3 host matrix: three sequential h2d calls
(row offsets, column indices narrowed, values) vs one interleaved
h2d_multi pass (what sparse.upload_csr does)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200._device import h2d, h2d_multi, warm_transfers

A = pb.stencil_device("3d7", int(sys.argv[1]) if len(sys.argv) > 1 else 256).to_host()
n, nnz = A.n_rows, int(A.row_offsets[-1])
warm_transfers()
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
col = torch.empty(nnz, dtype=torch.int32, device="cuda")
val = torch.empty(nnz, dtype=torch.float64, device="cuda")
def seq():
    h2d(rp, A.row_offsets, narrow=True); h2d(col, A.col_indices, narrow=True); h2d(val, A.values)
def multi():
    h2d_multi([(rp, A.row_offsets, True), (col, A.col_indices, True), (val, A.values, False)])
for rep in range(3):
    for name, fn in (("sequential", seq), ("interleaved", multi)):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
        print(f"{name}: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
