"""Summarise an ncu launch list (+ optional --set full report) into markdown.

    python tools/ncu_summary.py gpurun_out/launches.csv [gpurun_out/prof.ncu-rep] \
        --bytes <algorithmic bytes per launch of the top kernel> > profiles/rNN_x.md
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess

RAW_KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_selected",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    return agg


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    res = []
    for row in r[2:]:
        res.append({k: (row[h.index(k)], u[h.index(k)]) for k in RAW_KEYS if k in h}
                   | {"Kernel Name": (row[h.index("Kernel Name")], "")})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("launch_csv")
    ap.add_argument("report", nargs="?")
    ap.add_argument("--bytes", type=float, default=None)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--traffic-key", default=None,
                    help="'<bench config>/<engine code>': record the captured kernel's DRAM "
                         "bytes per launch in profiles/traffic.json (read by bench.py)")
    ap.add_argument("--source", default=None, help="profile file name recorded as the source")
    a = ap.parse_args()
    agg = launches(a.launch_csv)
    tot = sum(sum(v) for v in agg.values())
    print(f"# {a.title}\n")
    print("## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; "
          "cold-cache, serialised: compare shares)\n")
    print("| launches | total us | share | avg us | kernel |\n|---:|---:|---:|---:|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {len(v)} | {sum(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% | "
              f"{sum(v) / len(v) / 1e3:.1f} | `{k[:110]}` |")
    if a.report:
        per_launch = []  # (dram bytes, seconds, kernel) of every captured launch
        for rec in raw(a.report):
            print(f"\n## ncu --set full: `{rec['Kernel Name'][0][:120]}`\n")
            print("| metric | value | unit |\n|---|---:|---|")
            for k in RAW_KEYS:
                if k in rec:
                    print(f"| {k} | {rec[k][0]} | {rec[k][1]} |")
            try:
                t_us = float(rec["gpu__time_duration.sum"][0].replace(",", ""))
                unit = rec["gpu__time_duration.sum"][1]
                t_s = t_us * (1e-6 if unit == "us" else 1e-9 if unit == "ns" else 1e-3)
                rd = float(rec["dram__bytes_read.sum"][0].replace(",", ""))
                wr = float(rec["dram__bytes_write.sum"][0].replace(",", ""))
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
                rd *= scale[rec["dram__bytes_read.sum"][1]]
                wr *= scale[rec["dram__bytes_write.sum"][1]]
                print(f"\nDRAM traffic per launch: {(rd + wr) / 1e9:.4f} GB "
                      f"({(rd + wr) / t_s / 1e9:.0f} GB/s over the ncu duration)")
                per_launch.append((rd + wr, t_s, rec["Kernel Name"][0][:120]))
                if a.bytes:
                    print(f"Algorithmic (canonical) bytes per launch: {a.bytes / 1e9:.4f} GB; "
                          f"traffic/algorithmic = {(rd + wr) / a.bytes:.3f}")
            except (KeyError, ValueError):
                pass
        if per_launch:
            n = len(per_launch)
            avg_b = sum(p[0] for p in per_launch) / n
            avg_t = sum(p[1] for p in per_launch) / n
            if n > 1:
                print(f"\n## Average over the {n} captured launches (e.g. an even + an odd "
                      f"iteration of the deferred-x kernels)\n\nDRAM traffic per launch: "
                      f"{avg_b / 1e9:.4f} GB, {avg_t * 1e6:.1f} us, {avg_b / avg_t / 1e9:.0f} GB/s")
                if a.bytes:
                    print(f"traffic/algorithmic = {avg_b / a.bytes:.3f}")
            if a.traffic_key:
                import json
                import pathlib

                tp = pathlib.Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
                d = json.loads(tp.read_text()) if tp.exists() else {}
                d[a.traffic_key] = {"dram_bytes_per_launch": avg_b, "launches_averaged": n,
                                    "kernel": per_launch[0][2], "ncu_duration_s": avg_t,
                                    "source": a.source or a.report}
                tp.write_text(json.dumps(d, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
