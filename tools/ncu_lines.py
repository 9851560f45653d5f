"""Warp-stall samples per CUDA source line from an ncu report (source page, cuda,sass).

    python tools/ncu_lines.py gpurun_out/prof_x.ncu-rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, agg, srcs, hdr = None, {}, {}, None
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) >= 5 and r[0].strip():
        try:
            s = float(r[4] or 0)
        except ValueError:
            continue
        key = (cur, int(r[0]))
        agg[key] = agg.get(key, 0) + s
        srcs[key] = r[1]
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]:<5} {srcs[k][:100]}")
