import sys, time, ctypes, os
sys.path.insert(0, ".")
import torch, numpy as np
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200 import _lib, sparse as SP
path = sys.argv[1]
pb.load_matrix_market(path)
L = _lib.load()
for _ in range(2):
    t0 = time.perf_counter()
    h = ctypes.c_void_p(); rc = L.pipecg_b200_mm_read(os.fsencode(path), ctypes.byref(h)); t1 = time.perf_counter()
    A = SP._mm_csr(h); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"parse(host) {t1-t0:.3f}s  csr(device)+to_host+validate {t2-t1:.3f}s")
    d = A._b200_device[0]
    t3 = time.perf_counter(); B = d.to_host(); t4 = time.perf_counter()
    print(f"  to_host alone {t4-t3:.3f}s")
