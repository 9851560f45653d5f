"""Matrix Market ingestion throughput.

    python tools/mm_bench.py write /tmp/lap.mtx 3d7 128   # symmetric lower-triangle file
    python tools/mm_bench.py native /tmp/lap.mtx          # this repo (GPU box)
    PYTHONPATH=/root/reference/pkg/src python tools/mm_bench.py reference /tmp/lap.mtx  # dev container
"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

mode, path = sys.argv[1], sys.argv[2]
if mode == "write":
    import numpy as np
    import oracle

    S = oracle.stencil(sys.argv[3], int(sys.argv[4]))
    rows = np.repeat(np.arange(S.n_rows), np.diff(S.row_offsets))
    low = rows >= S.col_indices
    r, c, v = rows[low] + 1, S.col_indices[low] + 1, S.values[low]
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        f.write(f"{S.n_rows} {S.n_cols} {r.size}\n")
        step = 1 << 20
        for k in range(0, r.size, step):
            f.write("\n".join(f"{a} {b} {x:.17g}" for a, b, x in
                              zip(r[k:k + step].tolist(), c[k:k + step].tolist(),
                                  v[k:k + step].tolist())) + "\n")
    print(f"wrote {path}: {os.path.getsize(path) / 1e6:.1f} MB, {r.size} entries, nnz {S.nnz}")
    sys.exit(0)
size = os.path.getsize(path)
if mode == "native":
    import torch
    import paper_2105_06176_b200 as pb

    pb.load_matrix_market(path)  # warm (CUDA context, kernels)
    t = time.perf_counter()
    A = pb.load_matrix_market(path)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
else:
    from pipecg.sparse import load_matrix_market

    t = time.perf_counter()
    A = load_matrix_market(path)
    dt = time.perf_counter() - t
print(f"{mode}: {dt:.3f} s, {size / dt / 1e6:.1f} MB/s, {A.nnz / dt / 1e6:.2f} M nnz/s "
      f"(N={A.n_rows}, nnz={A.nnz}, cores={os.cpu_count()})")
