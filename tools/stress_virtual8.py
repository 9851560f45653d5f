"""Stress the 8-virtual-rank harness (threads sharing GPU 0): repeat the
world-8 solves of tests/test_gpu_distributed.py and count exchange
timeouts, optionally under memory pressure (argv[1] = GB held by torch)."""
import gc, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import torch
import paper_2105_06176_b200 as pb
from paper_2105_06176_b200 import distributed as D
import test_gpu_distributed as T

hold = None
if len(sys.argv) > 1 and float(sys.argv[1]) > 0:
    hold = torch.empty(int(float(sys.argv[1]) * 2**30), dtype=torch.uint8, device="cuda")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = pb.SolverConfig(tolerance=1e-9, max_iterations=3000, record_history=True)
cases = [(8, "3d7", 48, "fused-e"), (8, "3d7", 40, "fused-a"), (8, "3d27", 24, "fused-f"),
         (8, "3d7", 40, "fused-c")]
fails = 0
t0 = time.time()
for r in range(reps):
    for world, kind, n, eng in cases:
        out, errs = T._run_virtual_once(world, lambda g: D.shard_stencil(kind, n, g), cfg, 0, eng)
        if errs:
            fails += 1
            print(f"rep {r} {kind}-{n} {eng}: {errs[0][1][:220]}", flush=True)
        gc.collect()
print(f"{fails} failures in {reps * len(cases)} solves, {time.time() - t0:.0f} s", flush=True)
