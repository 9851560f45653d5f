"""Top SASS lines by warp-stall samples from an ncu report (source page).

    python tools/ncu_src_top.py gpurun_out/prof_x.ncu-rep [N]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
tot = sum(float(r[i_s] or 0) for r in data)
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:top_n]:
    print(f"{float(r[i_s]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[i_src][:100]}")
