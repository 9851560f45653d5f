"""Matrix Market ingestion vs the reference parser
(sparse.py:195-326).

* oracle/oracle.py's restatement is pinned to the reference's own outputs
  (tests/golden/mm_golden.*, made by importing the reference);
* the native parser (csrc/mmio.cu) must raise the same MatrixMarketError
  (message and 1-based line) on every malformed document -- host-side, so
  these run on CPU -- and build bitwise-identical CSR on the GPU.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

pb = pytest.importorskip("paper_2105_06176_b200")

CASES = json.loads((GOLDEN / "mm_golden.json").read_text())
ARR = np.load(GOLDEN / "mm_golden.npz")
OK = [k for k, v in CASES.items() if v["ok"]]
BAD = [k for k, v in CASES.items() if not v["ok"]]
H = "%%MatrixMarket matrix coordinate real general\n"


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(name):
    c = CASES[name]
    if c["ok"]:
        A = oracle.parse_matrix_market(c["text"].replace("\r\n", "\n"))
        np.testing.assert_array_equal(A.row_offsets, ARR[name + "_ro"])
        np.testing.assert_array_equal(A.col_indices, ARR[name + "_ci"])
        np.testing.assert_array_equal(A.values, ARR[name + "_va"])
    else:
        with pytest.raises(oracle.MMError) as e:
            oracle.parse_matrix_market(c["text"])
        assert (str(e.value), e.value.line_number) == (c["message"], c["line"])


@pytest.mark.parametrize("name", BAD)
def test_native_errors_match_reference(name):
    c = CASES[name]
    with pytest.raises(pb.MatrixMarketError) as e:
        pb.parse_matrix_market(c["text"])
    assert e.value.line_number == c["line"]
    assert str(e.value) == c["message"]
    assert isinstance(e.value, ValueError)


def _big_doc(rng, n_rows, n_entries, bad_at=None, bad_line="1 2 3 4"):
    rows = rng.integers(1, n_rows + 1, size=n_entries)
    cols = rng.integers(1, n_rows + 1, size=n_entries)
    vals = rng.standard_normal(n_entries)
    body = [f"{r} {c} {v!r}" for r, c, v in zip(rows.tolist(), cols.tolist(), vals.tolist())]
    for k in range(0, n_entries, 997):
        body[k] += "\n% comment\n"
    if bad_at is not None:
        body[bad_at] = bad_line
    return H + f"{n_rows} {n_rows} {n_entries}\n" + "\n".join(body) + "\n"


@pytest.mark.parametrize("bad_at,bad_line", [(5, "1 2"), (120_000, "x 1 1.0"),
                                               (239_999, "1 1 nope"), (150_000, "999999 1 1.0")])
def test_native_multichunk_error_order(bad_at, bad_line):
    """~6 MB documents split across threads: the first error in document
    order is the one reported, with its global line number."""
    text = _big_doc(np.random.default_rng(bad_at), 50_000, 240_000, bad_at, bad_line)
    with pytest.raises(oracle.MMError) as ref:
        oracle.parse_matrix_market(text)
    with pytest.raises(pb.MatrixMarketError) as got:
        pb.parse_matrix_market(text)
    assert (str(got.value), got.value.line_number) == (str(ref.value), ref.value.line_number)


def test_native_multichunk_count_errors():
    rng = np.random.default_rng(7)
    good = _big_doc(rng, 20_000, 200_000)
    lines = good.split("\n")
    more = "\n".join([lines[0], lines[1].replace("200000", "199990")] + lines[2:])
    less = "\n".join([lines[0], lines[1].replace("200000", "200005")] + lines[2:])
    for text in (more, less):
        with pytest.raises(oracle.MMError) as ref:
            oracle.parse_matrix_market(text)
        with pytest.raises(pb.MatrixMarketError) as got:
            pb.parse_matrix_market(text)
        assert (str(got.value), got.value.line_number) == (str(ref.value), ref.value.line_number)


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(OSError):
        pb.load_matrix_market(tmp_path / "nope.mtx")


# ---- GPU: CSR assembly on the device ------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", OK)
def test_native_csr_bitwise_vs_reference(cuda, name):
    A = pb.parse_matrix_market(CASES[name]["text"])
    assert [A.n_rows, A.n_cols] == CASES[name]["shape"]
    np.testing.assert_array_equal(A.row_offsets, ARR[name + "_ro"])
    np.testing.assert_array_equal(A.col_indices, ARR[name + "_ci"])
    np.testing.assert_array_equal(A.values, ARR[name + "_va"])


@pytest.mark.gpu
@pytest.mark.parametrize("newline", ["\n", "\r\n", "\r"])
def test_native_file_multichunk_vs_oracle(cuda, tmp_path, newline):
    text = _big_doc(np.random.default_rng(11), 3_000, 300_000)  # many duplicates
    p = tmp_path / "big.mtx"
    p.write_bytes(text.replace("\n", newline).encode())
    A = pb.load_matrix_market(p)
    R = oracle.parse_matrix_market(text)
    np.testing.assert_array_equal(A.row_offsets, R.row_offsets)
    np.testing.assert_array_equal(A.col_indices, R.col_indices)
    np.testing.assert_array_equal(A.values, R.values)


@pytest.mark.gpu
def test_loaded_matrix_solves_like_oracle(cuda, tmp_path):
    """File -> device CSR (kept resident) -> PIPECG, bitwise in seq mode."""
    S = oracle.stencil("3d7", 12)
    ro, ci, va = S.row_offsets, S.col_indices, S.values
    rows = np.repeat(np.arange(S.n_rows), np.diff(ro))
    low = rows >= ci
    lines = [f"{r + 1} {c + 1} {v!r}" for r, c, v in
             zip(rows[low].tolist(), ci[low].tolist(), va[low].tolist())]
    p = tmp_path / "lap.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n"
                 f"{S.n_rows} {S.n_cols} {len(lines)}\n" + "\n".join(lines) + "\n")
    A = pb.load_matrix_market(p)
    np.testing.assert_array_equal(A.col_indices, ci)
    np.testing.assert_array_equal(A.values, va)
    x_true, b, x0, d = oracle.manufactured(S)
    tol = oracle.recipe_tolerance(S, b, d)
    ref = oracle.pipecg_solve(S, b, x0, d, tol=tol, max_iterations=5000)
    cfg = pb.SolverConfig(tolerance=tol, max_iterations=5000, record_history=True)
    x, rep = pb.pipecg_solve(A, b, x0, pb.jacobi_setup(A), cfg,
                             options=pb.DeviceOptions(dot_mode="seq"))
    assert rep.history == ref.history
    np.testing.assert_array_equal(x, ref.x)
