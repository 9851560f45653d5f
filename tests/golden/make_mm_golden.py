"""Matrix Market golden cases, produced by the
reference parser itself (sparse.py:195-326).  Dev-container only: imports
/root/reference; the GPU box uses the committed tests/golden/mm_golden.*.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_mm_golden.py
"""
import json
from pathlib import Path

import numpy as np
from pipecg.sparse import MatrixMarketError, parse_matrix_market

OUT = Path(__file__).resolve().parent
H = "%%MatrixMarket matrix coordinate real "


def random_doc(rng, n_rows, n_cols, n, symmetric=False, crlf=False, comments=True):
    lines = [H + ("symmetric" if symmetric else "general"), "% generated"]
    if comments:
        lines.append("")
    lines.append(f"{n_rows} {n_cols} {n}")
    fmts = ["{:.17g}", "{:.6e}", "{:.3f}", "{:.17g}".replace("g", "G"), "{}"]
    for k in range(n):
        i = int(rng.integers(1, n_rows + 1))
        j = int(rng.integers(1, (i if symmetric else n_cols) + 1))
        v = float(rng.standard_normal() * 10.0 ** int(rng.integers(-5, 5)))
        s = fmts[k % len(fmts)].format(v)
        if k % 7 == 3:
            s = s.replace("e", "d") if "e" in s else s  # Fortran exponent
        if k % 11 == 5:
            s = "+" + s.lstrip("+") if not s.startswith("-") else s
        lines.append(f"{i} {j} {s}" if k % 5 else f"  {i}\t{j}   {s}  ")
        if comments and k % 13 == 0:
            lines.append("% mid comment")
        if comments and k % 17 == 0:
            lines.append("   ")
    sep = "\r\n" if crlf else "\n"
    return sep.join(lines) + sep


def main():
    rng = np.random.default_rng(20261017)
    docs = {
        "general_dups": random_doc(rng, 40, 55, 900),  # many duplicate coordinates
        "symmetric": random_doc(rng, 60, 60, 700, symmetric=True),
        "crlf": random_doc(rng, 30, 30, 300, crlf=True),
        "heavy_dups": random_doc(rng, 2, 3, 1500),  # 250 per coordinate: pairwise blocks
        "mid_dups": random_doc(rng, 4, 5, 200),     # ~10 per coordinate
        "underscores": H + "general\n3 3 4\n1 1 1_000.5\n2 2 -2.5E+0_1\n3 1 .5\n1_0 3 5.\n".replace("1_0 3", "3 3"),
        "inf_nan_big": H + "general\n2 2 4\n1 1 inf\n1 2 -Infinity\n2 1 1e400\n2 2 4.9e-324\n",
        "header_case": "%%matrixmarket MATRIX Coordinate REAL General extra tokens\n1 2 2\n1 2 3.0\n1 1 1D-3\n",
    }
    # malformed documents (reference tests/test_sparse.py:152-180 style + more)
    bad = {
        "empty": "",
        "hdr": "%%NotMatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n",
        "object": "%%MatrixMarket tensor coordinate real general\n1 1 1\n1 1 1.0\n",
        "format": "%%MatrixMarket matrix array real general\n1 1 1\n1 1 1.0\n",
        "field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0\n",
        "symmetry": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1.0\n",
        "nosize": H + "general\n% only comments\n",
        "size2": H + "general\n2 2\n",
        "sizex": H + "general\n2 2 x\n",
        "size0": H + "general\n2 2 0\n",
        "symsq": H + "symmetric\n2 3 1\n1 1 1.0\n",
        "rowoob": H + "general\n2 2 1\n3 1 1.0\n",
        "coloob": H + "general\n2 2 1\n1 0 1.0\n",
        "coord": H + "general\n2 2 1\na 1 1.0\n",
        "value": H + "general\n2 2 1\n1 1 abc\n",
        "fields": H + "general\n2 2 1\n1 1\n",
        "excess": H + "general\n1 1 1\n1 1 1.0\n1 1 2.0\n",
        "excess_bad": H + "general\n1 1 1\n1 1 1.0\n1 1 zzz\n",
        "short": H + "general\n2 2 3\n1 1 1.0\n2 2 2.0\n",
        "short_comments": H + "general\n2 2 3\n1 1 1.0\n% c\n\n2 2 2.0\n% tail\n",
        "neg_row": H + "general\n2 2 1\n-1 1 1.0\n",
        "big_row": H + "general\n2 2 1\n123456789012345678901234 1 1.0\n",
        "quote_value": H + "general\n2 2 1\n1 1 it's\n",
        "late_error": random_doc(np.random.default_rng(3), 50, 50, 400, comments=False).replace(
            "\n", "\n", 1)[:-1] + "\n1 2 3 4\n",
    }
    # make late_error consistent: declare one more entry so the bad line is reached
    d = bad["late_error"].split("\n")
    d[1] = "50 50 401"
    bad["late_error"] = "\n".join(d)
    cases = {}
    arrays = {}
    for name, text in {**docs, **bad}.items():
        try:
            A = parse_matrix_market(text)
            cases[name] = {"ok": True, "shape": [A.n_rows, A.n_cols], "nnz": A.nnz}
            arrays[name + "_ro"] = A.row_offsets
            arrays[name + "_ci"] = A.col_indices
            arrays[name + "_va"] = A.values
        except MatrixMarketError as e:
            cases[name] = {"ok": False, "line": e.line_number, "message": str(e)}
        cases[name]["text"] = text
    (OUT / "mm_golden.json").write_text(json.dumps(cases, indent=1))
    np.savez_compressed(OUT / "mm_golden.npz", **arrays)
    print({k: (v["ok"], v.get("line")) for k, v in cases.items()})


if __name__ == "__main__":
    main()
