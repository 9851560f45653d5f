"""Time the fused iteration kernel under plan/flag overrides (experiments)."""
import math, os, sys, json
sys.path.insert(0, '.')
import torch
import paper_2105_06176_b200 as pb

def time_variant(A, d, env, steps=100, warm=5):
    for k in ("PIPECG_B200_TR", "PIPECG_B200_STAGES", "PIPECG_B200_BPS", "PIPECG_B200_FLAGS"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    N = A.n_rows
    xt = torch.full((N,), 1 / math.sqrt(N), dtype=torch.float64, device="cuda")
    b = pb.spmv(A, xt)
    try:
        s = pb.PipecgSolver(A, d)
    except Exception as e:
        return {"env": env, "error": str(e)[:200]}
    s.init(b, torch.zeros_like(b), 0.0, warm + steps + 1)
    s.enqueue(warm)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(s.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.enqueue(steps); e1.record(st); e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    s.close()
    return {"env": env, "ms": round(ms, 4)}

if __name__ == "__main__":
    kind, n = sys.argv[1], int(sys.argv[2])
    variants = json.loads(sys.argv[3])
    A = pb.stencil_device(kind, n)
    d = pb.jacobi_setup(A).inv_diag
    N, nnz = A.n_rows, A.nnz
    B = 176 * N + 12 * nnz + 4 * (N + 1)
    actual = 136 * N + 12 * nnz + 4 * (N + 1)
    for v in variants:
        r = time_variant(A, d, v)
        if "ms" in r:
            r["canon_GBs"] = round(B / r["ms"] / 1e6)
            r["actual_GBs"] = round(actual / r["ms"] / 1e6)
        print(json.dumps(r), flush=True)
