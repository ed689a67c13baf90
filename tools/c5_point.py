#!/usr/bin/env python
"""Run one c5 microbench point (standalone NTT fwd / inv or MAC) a few times -- the
command ncu profiles.  Prints the CUDA-event time and GB/s of the last repetitions.

usage: python tools/c5_point.py --lg 13 --L 9 --bits 48 --op fwd [--batch B] [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lg", type=int, default=13)
    ap.add_argument("--L", type=int, default=9)
    ap.add_argument("--bits", type=int, default=48)
    ap.add_argument("--op", default="fwd", choices=["fwd", "inv", "mac"])
    ap.add_argument("--batch", type=int, default=0, help="polynomials (0: a 2 GiB working set)")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--alt-teams", action="store_true")
    ap.add_argument("--u32", action="store_true", help="u32 words (30-bit primes): ephdc_ntt_fwd32 / inv32")
    ap.add_argument("--u32-generic", action="store_true", help="with --u32: the general u32 kernels")
    a = ap.parse_args()
    import torch
    import paper_2511_00737_b200 as eph

    N = 1 << a.lg
    q = eph.find_ntt_primes(a.lg, [a.bits] * a.L)
    plan = eph.NttPlan(q, a.lg, alt_teams=a.alt_teams, u32_generic=a.u32_generic)
    wb = 4 if a.u32 else 8
    per_poly = a.L * N * wb
    dev = torch.device("cuda", 0)
    qt = torch.tensor(q, dtype=torch.int64, device=dev)
    if a.op == "mac":
        D = a.batch or max(1, (2 << 30) // (3 * per_poly))
        ct = torch.remainder(torch.randint(0, 1 << 62, (D, a.L, 2, N), dtype=torch.int64, device=dev), qt.view(1, -1, 1, 1))
        pt = torch.remainder(torch.randint(0, 1 << 62, (D, a.L, N), dtype=torch.int64, device=dev), qt.view(1, -1, 1))
        out = torch.empty((a.L, 2, N), dtype=torch.int64, device=dev)
        fn = lambda: eph.mac(plan, ct, pt, out)  # noqa: E731
        nbytes = 3 * D * per_poly
    else:
        batch = a.batch or max(1, (2 << 30) // per_poly)
        x = torch.remainder(torch.randint(0, 1 << 62, (batch, a.L, N), dtype=torch.int64, device=dev), qt.view(1, -1, 1))
        if a.u32:
            x = x.to(torch.int32)
            f = eph.ntt_fwd32 if a.op == "fwd" else eph.ntt_inv32
        else:
            f = eph.ntt_fwd if a.op == "fwd" else eph.ntt_inv
        fn = lambda: f(plan, x)  # noqa: E731
        nbytes = 2 * batch * per_poly
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(json.dumps({"lg": a.lg, "L": a.L, "bits": a.bits, "op": a.op, "ms": round(ms, 4),
                      "GB_s": round(nbytes / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
