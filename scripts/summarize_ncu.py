"""Summaries of ncu outputs for profiles/ (launch lists and --set full reports)."""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    data = collections.OrderedDict()
    for r in rows:
        data.setdefault(r[ii], {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    out = ["| # | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | GB/s |", "|---|---|---|---|---|---|"]
    for i, d in data.items():
        t = d.get("gpu__time_duration.sum", 0.0)
        rb, wb = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        name = d["k"].split("(")[0].replace("void ", "")[-48:]
        out.append(f"| {i} | `{name}` | {t / 1e3:.1f} | {rb / 1e6:.1f} | {wb / 1e6:.1f} | {(rb + wb) / t if t else 0:.0f} |")
    return "\n".join(out)


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    out = []
    for v in vals:
        out.append(f"kernel: {v[hdr.index('Kernel Name')]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k} = {v[i]} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
