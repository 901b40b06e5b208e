#!/usr/bin/env python
"""Summarise ncu output for profiles/ (run here, on the CPU box).

    python scripts/summarize_ncu.py launches gpurun_out/launches.csv > profiles/r01_launches.md
    python scripts/summarize_ncu.py full gpurun_out/prof.ncu-rep > profiles/r01_full.md
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = []
    with open(path) as f:
        text = f.read()
    # ncu --csv --log-file: header line starts with "ID"
    start = text.find('"ID"')
    rdr = csv.DictReader(io.StringIO(text[start:]))
    for r in rdr:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "")
            us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
            rows.append((int(r["ID"]), r["Kernel Name"].split("(")[0], us))
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for _, k, us in rows:
        tot[k] = tot.get(k, 0.0) + us
        cnt[k] += 1
    T = sum(tot.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    print(f"{len(rows)} launches, {T/1000:.3f} ms total\n")
    print("| kernel | launches | total us | share | mean us |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v:.1f} | {v / T:.1%} | {v / cnt[k]:.1f} |")


FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__cluster_dim_x", "smsp__cycles_active.avg",
    "sm__cycles_elapsed.avg.per_second",
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("# ncu --set full summary (one capture per listed launch)\n")
    cols = [m for m in FULL_METRICS if m in hdr]
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        vals = [f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip() for m in cols]
        print(f"| {name} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
