#!/usr/bin/env python
"""Summarise ncu output for profiles/: the launch list (per-kernel count, total and
mean device time, share) and the key metrics of a `--set full` capture.

usage: python tools/ncu_summary.py launches <launches.csv>
       python tools/ncu_summary.py full <prof.ncu-rep>
"""
import collections
import csv
import io
import re
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        ms = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'total_ms':>11s} {'mean_ms':>10s} {'share':>7s}")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:44s} {n:8d} {t:11.3f} {t / n:10.4f} {t / tot:7.3f}")


KEYS = [r"gpu__time_duration.sum$", r"dram__bytes_(read|write)\.sum$", r"launch__registers_per_thread$",
        r"launch__shared_mem_per_block$", r"launch__occupancy_limit_(registers|shared_mem|warps)$",
        r"sm__warps_active.avg.pct_of_peak_sustained_active$", r"sm__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed$", r"dram__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"lts__throughput.avg.pct_of_peak_sustained_elapsed$", r"l1tex__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"sm__pipe_(alu|fma|fmaheavy|fp64|shared|tensor)_cycles_active.avg.pct_of_peak_sustained_elapsed$",
        r"sm__inst_executed_pipe_(alu|fma|fmaheavy|fmalite|fp64|lsu|uniform|xu)\.avg.pct_of_peak_sustained_active$",
        r"smsp__issue_active.avg.pct_of_peak_sustained_active$",
        r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$",
        r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared.*sum$", r"smsp__inst_executed.sum$",
        r"lts__t_sector_hit_rate.pct$"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    pats = [re.compile(k) for k in KEYS]
    for r in rows[2:]:
        kn = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"== {kn[:100]}")
        for i, name in enumerate(h):
            if any(p.search(name) for p in pats):
                v = r[i]
                if name.startswith("smsp__average_warps_issue_stalled"):
                    try:
                        if float(v) < 0.05:
                            continue
                    except ValueError:
                        pass
                print(f"  {name:80s} {u[i]:>12s} {v}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
