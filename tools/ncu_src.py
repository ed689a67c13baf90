#!/usr/bin/env python
"""Summarise an ncu report's SASS source page: instruction mix by opcode and the
hottest instructions by stall samples.  usage: ncu_src.py <rep> [kernel-substring] [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    ops = collections.Counter()
    stalls = collections.Counter()
    tot = 0.0
    for r in data:
        src = r[iSrc].strip()
        parts = src.split()
        op = parts[1] if parts and parts[0].startswith("@") and len(parts) > 1 else (parts[0] if parts else "?")
        op = op.split(".")[0]
        n = float(r[iE] or 0)
        ops[op] += n
        stalls[op] += float(r[iS] or 0)
        tot += n
    print(f"total warp-instructions {tot:.4g}")
    for op, n in ops.most_common(30):
        print(f"  {op:12s} {n:12.4g} {100 * n / tot:5.1f}%  stall-samples {stalls[op]:.0f}")
    print("-- hottest by stall samples")
    for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:top]:
        print(f"  {r[0][-5:]} {r[iS]:>7} {r[iE]:>10}  {r[iSrc].strip()[:90]}")


if __name__ == "__main__":
    main()
