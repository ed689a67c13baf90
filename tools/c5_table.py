#!/usr/bin/env python
"""Summarise a tools/bench_c5.py sweep (one JSON line per point and batch) as the
BASELINE.md table: forward / inverse fraction of the measured HBM bandwidth at the
largest batch of each (N, prime class, word) -- the best L -- with the median SM clock
and any throttle reason of that line.  Reads only the committed .jsonl; measures nothing.

usage: python tools/c5_table.py profiles/r02/r67/c5_all.jsonl
"""
from __future__ import annotations

import json
import sys


def main():
    rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip().startswith("{")]
    ntt = [r for r in rows if "ntt_fwd" in r]
    mac = [r for r in rows if r.get("op") == "mac"]
    classes = [(48, 64), (30, 64), (30, 32), (60, 64)]
    print("| N | " + " | ".join(f"{b}-bit, u{w}" for b, w in classes) + " |")
    print("|---|" + "---|" * len(classes))
    for lg in sorted({r["log2N"] for r in ntt}):
        cells = []
        for b, w in classes:
            pts = [r for r in ntt if r["log2N"] == lg and r["bits"] == b and r["word_bits"] == w]
            if not pts:
                cells.append("-")
                continue
            bmax = max(r["batch"] for r in pts)
            best = max((r for r in pts if r["batch"] == bmax),
                       key=lambda r: r["ntt_fwd"]["frac_hbm"] + r["ntt_inv"]["frac_hbm"])
            c = best["clocks"]
            note = f"L={best['L']}, batch {bmax}, {c['sm_mhz']:.0f} MHz"
            if c.get("reasons"):
                note += ", " + "+".join(c["reasons"])
            k = best.get("kernels", {})
            cells.append(f"{best['ntt_fwd']['frac_hbm']:.2f} / {best['ntt_inv']['frac_hbm']:.2f} "
                         f"({k.get('fwd', '?')}/{k.get('inv', '?')}; {note})")
        print(f"| 2^{lg} | " + " | ".join(cells) + " |")
    if mac:
        print()
        print("| MAC class | min .. max fraction of HBM over the points |")
        print("|---|---|")
        for b, w in classes:
            pts = [r for r in mac if r["bits"] == b and r["word_bits"] == w]
            if pts:
                fr = [r["frac_hbm"] for r in pts]
                print(f"| {b}-bit, u{w} | {min(fr):.2f} .. {max(fr):.2f} ({len(pts)} points) |")
    bad = [r for r in rows if not r.get("clocks") or r["clocks"].get("samples", 0) == 0]
    print(f"\n{len(rows)} lines, {len(bad)} without a clock record")


if __name__ == "__main__":
    main()
