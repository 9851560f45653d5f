"""Time PIPECG iterations under engine/plan choices (same box, same binary).

    python tools/sweep.py 3d7 256 '[{"engine": "fused-a"}, {"engine": "fused-b"}, {"engine": "two"}]'
Keys other than DeviceOptions fields are set as environment variables
(PIPECG_B200_STAGES / _TR / _FLAGS experiment overrides)."""
import math, os, sys, json
sys.path.insert(0, '.')
import torch
import paper_2105_06176_b200 as pb

OPT_KEYS = {"engine", "dot_mode", "chunk", "use_graphs", "max_sms"}

def time_variant(A, d, v, steps=40, warm=5):
    for k in list(os.environ):
        if k.startswith("PIPECG_B200_"):
            os.environ.pop(k)
    os.environ.update({k: str(x) for k, x in v.items() if k not in OPT_KEYS})
    opts = pb.DeviceOptions(**{k: x for k, x in v.items() if k in OPT_KEYS})
    N = A.n_rows
    xt = torch.full((N,), 1 / math.sqrt(N), dtype=torch.float64, device="cuda")
    b = pb.spmv(A, xt)
    try:
        s = pb.PipecgSolver(A, d, opts)
    except Exception as e:
        return {"v": v, "error": str(e)[:200]}
    s.init(b, torch.zeros_like(b), 0.0, warm + steps + 1)
    s.enqueue(warm)
    s.prepare(steps)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(s.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.enqueue(steps); e1.record(st); e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    res = s.poll()
    s.close()
    return {"v": v, "ms": round(ms, 4), "engine": res.engine,
            "tune": [round(t, 4) for t in res.tune_ms]}

if __name__ == "__main__":
    kind, n = sys.argv[1], int(sys.argv[2])
    variants = json.loads(sys.argv[3])
    A = (pb.as_device_csr(pb.generate_powerlaw(2**n)) if kind == "powerlaw"
         else pb.stencil_device(kind, n))
    d = pb.jacobi_setup(A).inv_diag
    N, nnz = A.n_rows, A.nnz
    B = 176 * N + 12 * nnz + 4 * (N + 1)
    for v in variants:
        r = time_variant(A, d, v)
        if "ms" in r:
            r["canon_GBs"] = round(B / r["ms"] / 1e6)
        print(kind, n, json.dumps(r), flush=True)
