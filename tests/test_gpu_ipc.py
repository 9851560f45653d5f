"""The multi-PROCESS path (CUDA IPC-mapped peer memory, torch.distributed
setup) on one B200: two processes share cuda:0 (kernels of different
processes are time-sliced, so the in-kernel waits still make progress).
On a multi-GPU node the same code maps NVLink peer memory instead."""

from __future__ import annotations

import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, q):
    import torch.distributed as dist

    import paper_2105_06176_b200 as pb
    from paper_2105_06176_b200 import distributed as D

    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        g = D.TorchGroup()
        prob = D.shard_stencil(kind, n, g)
        xt, b = D.manufactured_local(prob)
        cfg = pb.SolverConfig(tolerance=1e-9, max_iterations=500, record_history=True)
        x, rep = D.pipecg_solve_distributed(prob, b, torch.zeros_like(b), cfg, g,
                                            pb.DeviceOptions(max_sms=60))
        q.put((rank, x.cpu().numpy(), rep.iterations, rep.history, None))
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        q.put((rank, None, None, None, repr(e)[:500]))


def test_two_processes_ipc(cuda):
    import torch.multiprocessing as mp

    kind, n, world = "3d7", 16, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, kind, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=120)
    errs = [r[4] for r in res if r[4]]
    assert not errs, errs
    A = oracle.stencil(kind, n)
    x_true, b, x0, d = oracle.manufactured(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=1e-9, max_iterations=500)
    x = np.concatenate([r[1] for r in res])
    assert res[0][2] == res[1][2]
    assert abs(res[0][2] - ref.iterations) <= 1
    assert oracle.history_gap(res[0][3], ref.history) <= 1e-10
    assert np.max(np.abs(x - ref.x)) / np.max(np.abs(ref.x)) <= 1e-8
