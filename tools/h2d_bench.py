"""Host->device pipeline throughput vs host threads (pageable numpy source)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2105_06176_b200._device import h2d, d2h, warm_transfers
n = 1 << 27  # 1 GiB of int64 / float64
a = np.arange(n, dtype=np.int64)
f = np.random.default_rng(0).standard_normal(n)
warm_transfers()
d32 = torch.empty(n, dtype=torch.int32, device="cuda")
d64 = torch.empty(n, dtype=torch.float64, device="cuda")
for name, fn in (("narrow i64->i32", lambda: h2d(d32, a, narrow=True)), ("copy f64", lambda: h2d(d64, f)),
                 ("torch pageable f64", lambda: d64.copy_(torch.from_numpy(f))),
                 ("d2h f64", lambda: d2h(d64))):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{name}: {8 * n / dt / 1e9:.1f} GB/s of host source ({dt * 1e3:.1f} ms)", flush=True)
t = time.perf_counter(); b = f.copy(); dt = time.perf_counter() - t
print(f"numpy 1-thread copy: {16 * n / dt / 1e9:.1f} GB/s (r+w)")
# d2h into an already-touched destination (page faults out of the picture)
from paper_2105_06176_b200 import _lib
from paper_2105_06176_b200._device import stream_ptr
out = np.ones(n)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    _lib.call("pipecg_b200_d2h", out.ctypes.data, d64.data_ptr(), out.nbytes, stream_ptr())
    torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"d2h f64 into touched pages: {8 * n / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
t = time.perf_counter(); z = np.empty(n); z[::512] = 0.0; dt = time.perf_counter() - t
print(f"first-touch 1 page in 4 (1 thread): {8 * n / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
