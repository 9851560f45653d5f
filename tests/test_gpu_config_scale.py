"""Config-scale parity: the engines the bench runs, at the sizes it quotes.

Goldens: tests/golden/config_scale/<config>.{json,npz}, written by
tests/golden/make_config_goldens.py from the oracle (the reference itself
pinned them bit for bit at 3D 7-pt 128^3 and 256^3: ``pinned_by_reference``).
Each case solves the recipe problem (x_true = 1/sqrt(N),
b = A x_true, x0 = 0, Jacobi, tol = 1e-8 sqrt((u0,u0)), max 20000) with the
matrix generated in HBM exactly as bench.py does, then applies BASELINE.md's
gates against the golden:

1. iterations within +-1;
2. G = max_k |h_k - h_k^ref| / h_0 <= max(1e-10, 3E), E the oracle's own
   dot-reorder envelope at that config (stored beside the history);
3. x within max(1e-8, 3 x-envelope) relative, on 65,536 strided samples;
4. dot_mode="seq": history and the whole x (sha256) bit for bit, for every
   configuration without hub rows, up to 256^3.

Engines: "auto" (what the bench's autotuner picks -- E at 7-pt, F at 27-pt,
the two-kernel SELL engine on the power-law graph) and each engine forced.
These are the grid / tile / plan shapes of the bench (444-CTA grids, 256-row
tiles, 3 CTAs per SM at 256^3), which the small-case tests never reach.
"""

from __future__ import annotations

import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

pb = pytest.importorskip("paper_2105_06176_b200")
torch = pytest.importorskip("torch")

GDIR = Path(__file__).resolve().parent / "golden" / "config_scale"
CONFIGS = sorted(p.stem for p in GDIR.glob("*.json"))

STENCIL_ENGINES = ["auto", "fused-e", "fused-f", "fused-a", "fused-c", "two"]
IRREGULAR_ENGINES = ["auto", "two", "fused-g", "fused-d"]
ENGINE_NAMES = {2: "two", 3: "fused-a", 4: "fused-b", 5: "fused-c", 6: "fused-d",
                7: "fused-p", 8: "fused-e", 9: "fused-f", 10: "fused-g"}


def meta(name):
    return json.loads((GDIR / f"{name}.json").read_text())


def golden(name):
    with np.load(GDIR / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


_PROBLEMS = {}


def problem(name):
    """Device matrix + recipe vectors, built as bench.py builds them."""
    if name in _PROBLEMS:
        return _PROBLEMS[name]
    _PROBLEMS.clear()
    torch.cuda.empty_cache()
    m = meta(name)
    if m["kind"] == "powerlaw":
        A = pb.as_device_csr(pb.generate_powerlaw(2 ** m["n"]))
    else:
        A = pb.stencil_device(m["kind"], m["n"])
    assert (A.n_rows, A.nnz) == (m["N"], m["nnz"])
    N = A.n_rows
    x_true = torch.full((N,), 1.0 / math.sqrt(N), dtype=torch.float64, device="cuda")
    b = pb.spmv(A, x_true)  # reference row order: bitwise the oracle's b
    pc = pb.jacobi_setup(A)
    u0 = pb.jacobi_apply(pc, b)
    tol = 1e-8 * math.sqrt(pb.dot(u0, u0, mode="seq"))
    _PROBLEMS[name] = (A, b, pc, tol)
    return _PROBLEMS[name]


def engine_used(A) -> str:
    s = next(iter(A.__dict__.get("_solvers", {}).values()), None)
    return ENGINE_NAMES.get(s.poll().engine, "?") if s is not None else "?"


def cases():
    out = []
    for name in CONFIGS:
        engines = IRREGULAR_ENGINES if name.startswith("powerlaw") else STENCIL_ENGINES
        out += [(name, e) for e in engines]
    return out


@pytest.mark.parametrize("name,engine", cases())
def test_config_scale_tree_gates(cuda, name, engine):
    m, g = meta(name), golden(name)
    A, b, pc, tol = problem(name)
    # the recipe tolerance is a function of b and inv_diag: equal bits mean
    # the device problem is the golden's problem
    assert tol == m["tol"], (tol, m["tol"])
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, torch.zeros_like(b), pc, cfg,
                             options=pb.DeviceOptions(engine=engine))
    used = engine_used(A)
    assert rep.converged
    assert abs(rep.iterations - m["iterations"]) <= 1, (used, rep.iterations, m["iterations"])
    G = oracle.history_gap(rep.history, list(g["history"]))
    assert G <= max(1e-10, 3 * m["E"]), (used, G, m["E"])
    idx = torch.as_tensor(g["x_idx"], device="cuda")
    xs = x[idx].cpu().numpy()
    ref = g["x_sample"]
    rel = float(np.max(np.abs(xs - ref)) / np.max(np.abs(ref)))
    assert rel <= max(1e-8, 3 * m["x_gap_blocked"]), (used, rel, m["x_gap_blocked"])
    print(f"{name} {engine}->{used}: it={rep.iterations} (golden {m['iterations']}) "
          f"G={G:.2e} (E={m['E']:.2e}) x_rel={rel:.2e}")


def seq_cases():
    out = []
    for name in CONFIGS:
        m = meta(name)
        if m["kind"] == "powerlaw" or m["N"] > 2 ** 24:
            continue  # hub rows are tree-combined; 400^3 seq dots take minutes
        # the sequential dots are one warp (~0.2 s per iteration at 256^3):
        # the bench's own engine there, every engine below
        engines = ["auto"] if m["N"] > 2 ** 22 else STENCIL_ENGINES
        out += [(name, e) for e in engines]
    return out


@pytest.mark.parametrize("name,engine", seq_cases())
def test_config_scale_seq_bitwise(cuda, name, engine):
    m, g = meta(name), golden(name)
    A, b, pc, tol = problem(name)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=20000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, torch.zeros_like(b), pc, cfg,
                             options=pb.DeviceOptions(engine=engine, dot_mode="seq"))
    used = engine_used(A)
    assert rep.iterations == m["iterations"], used
    np.testing.assert_array_equal(np.array(rep.history), g["history"])
    h = hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()
    assert h == m["x_sha256"], f"{name} {engine}->{used}: x differs from the reference"
