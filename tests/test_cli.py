"""The pipecg-bench front end on the B200 path:
same subcommands, run-record JSON, CSV columns and exit codes as the
reference (cli.py:49-54, 103-149, 227-255, 424-434)."""

from __future__ import annotations

import csv
import io
import json

import numpy as np
import pytest

import oracle

pb = pytest.importorskip("paper_2105_06176_b200")
from paper_2105_06176_b200 import cli  # noqa: E402

REFERENCE_CSV_COLUMNS = ["problem", "N", "nnz", "strategy", "iterations", "converged",
                         "final_norm", "wall_ms", "transfer_values", "verify_inf_err", "speedup"]


def test_csv_columns_are_the_references():
    assert cli.CSV_COLUMNS == REFERENCE_CSV_COLUMNS


def test_usage_errors_exit_1(capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["solve"])  # no problem source
    assert e.value.code == 1
    with pytest.raises(SystemExit) as e:
        cli.main(["solve", "--poisson", "6", "--stencil", "3d7-8"])  # two sources
    assert e.value.code == 1


def test_value_errors_exit_1(capsys):
    assert cli.main(["compare", "--stencil", "3d7-8", "--strategies", "nope"]) == 1
    assert cli.main(["compare", "--stencil", "3d7-8", "--strategies", "pipecg-b200",
                     "--baseline", "pcg-b200"]) == 1
    assert cli.main(["solve", "--stencil", "3d7-8", "--tol", "0"]) == 1
    assert "error:" in capsys.readouterr().err


def test_reference_command_line_flags_accepted():
    args = cli.build_parser().parse_args(
        ["solve", "--poisson", "6", "--host-workers", "4", "--accel-throttle", "2.0",
         "--xfer-latency-us", "5", "--pin-ratio", "0.3", "--seed", "1"])
    assert args.poisson == 6 and args.strategy == "pipecg-b200"


def test_run_record_round_trip():
    rep = pb.SolveReport(converged=True, iterations=3, final_norm=1e-9, strategy="pipecg",
                         history=[1.0, 0.1, 1e-9], phase_times={"setup": 0.1, "iterations": 0.2})
    rec = cli.RunRecord("p", "pipecg-b200", 10, 28, 1.5, "t", {"gpu": "B200"}, rep)
    back = cli.RunRecord.from_json(rec.to_json())
    assert back.to_dict() == rec.to_dict()


@pytest.mark.gpu
def test_solve_json_matches_oracle(cuda, capsys):
    rc = cli.main(["solve", "--stencil", "3d7-16", "--tol", "1e-9", "--history"])
    out = json.loads(capsys.readouterr().out)
    A = oracle.stencil("3d7", 16)
    x_true, b, x0, d = oracle.manufactured(A)
    ref = oracle.pipecg_solve(A, b, x0, d, tol=1e-9, max_iterations=10000)
    assert rc == 0
    assert out["strategy"] == "pipecg-b200" and out["n"] == A.n_rows and out["nnz"] == A.nnz
    assert abs(out["report"]["iterations"] - ref.iterations) <= 1
    assert out["report"]["verification_error"] < 1e-6
    assert len(out["report"]["history"]) == out["report"]["iterations"] + 1


@pytest.mark.gpu
def test_compare_csv_and_matrix_file(cuda, tmp_path, capsys):
    S = oracle.stencil("2d5", 30)
    rows = np.repeat(np.arange(S.n_rows), np.diff(S.row_offsets))
    lines = [f"{r + 1} {c + 1} {v!r}" for r, c, v in
             zip(rows.tolist(), S.col_indices.tolist(), S.values.tolist())]
    p = tmp_path / "lap2d.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n"
                 f"{S.n_rows} {S.n_cols} {len(lines)}\n" + "\n".join(lines) + "\n")
    rc = cli.main(["compare", "--matrix", str(p), "--tol", "1e-10",
                   "--strategies", "pcg-b200,pipecg-b200", "--baseline", "pcg-b200"])
    table = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    assert rc == 0
    assert [r["strategy"] for r in table] == ["pcg-b200", "pipecg-b200"]
    assert all(r["problem"] == "lap2d" and r["converged"] == "true" for r in table)
    assert float(table[0]["speedup"]) == 1.0
    assert abs(int(table[0]["iterations"]) - int(table[1]["iterations"])) <= 1


@pytest.mark.gpu
def test_exit_codes_nonconvergence_and_breakdown(cuda, tmp_path, capsys):
    assert cli.main(["solve", "--stencil", "3d7-16", "--tol", "1e-12", "--max-iters", "2"]) == 3
    p = tmp_path / "indef.mtx"  # diag(1, -1): alpha denominator breakdown at iteration 0
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2 -1.0\n")
    assert cli.main(["solve", "--matrix", str(p)]) == 2
    assert "alpha denominator" in capsys.readouterr().err
    rc = cli.main(["compare", "--matrix", str(p), "--strategies", "pipecg-b200",
                   "--format", "json"])
    rec = json.loads(capsys.readouterr().out)["records"][0]
    assert rc == 3 and rec["error"] and not rec["report"]["converged"]
