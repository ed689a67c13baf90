#!/usr/bin/env python
"""Stall samples and executed instructions per CUDA source line of an ncu report
(--page source --print-source cuda,sass; needs -lineinfo).  usage: ncu_lines.py <rep> [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = {}
    fname = "?"
    cur = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] == "Line No":
            continue
        if r[0]:   # a source line row (its metrics aggregate its SASS)
            cur = (fname, int(r[0]), r[1].strip()[:90])
            try:
                agg[cur] = (float(r[4] or 0), float(r[7] or 0))
            except ValueError:
                pass
    tot = sum(v[0] for v in agg.values()) or 1.0
    print(f"total stall samples {tot:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / tot:5.1f}% {v[1]:>11.4g}  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
