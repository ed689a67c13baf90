#!/usr/bin/env python
"""c5 kernel microbench (BASELINE.json configs[4]): standalone negacyclic NTT (forward,
inverse) and the pointwise ct x pt MAC on uniform residues, one JSON line per point.

GB/s = algorithmic bytes / CUDA-event time on the launching stream:
  NTT: read + write of batch x L x N u64 residues (in place);
  MAC: read of D x L x (2 + 1) x N u64 (two ciphertext residues + one plaintext).
Working sets are >= 1 GiB (8x L2) so every timed repetition streams from HBM.
Peak: MEASURED_PEAKS.json hbm_gbs.

usage: python tools/bench_c5.py [--points quick|all] [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", default="quick", choices=["quick", "all"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--bytes", type=float, default=2.0, help="GiB working set per point")
    a = ap.parse_args()
    import torch
    import ephdc_inputs as inp
    import paper_2511_00737_b200 as eph

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6460.5)
    if a.points == "quick":
        pts = [(lg, L, b) for lg in (12, 13, 14, 15, 16) for L, b in ((9, 48), (5, 60), (16, 30))]
    else:
        pts = [(lg, L, b) for lg in inp.C5_LOG2N for L in inp.C5_L for b in inp.C5_WORD_BITS]
    dev = torch.device("cuda", 0)
    for lg, L, bits in pts:
        N = 1 << lg
        q = eph.find_ntt_primes(lg, [bits] * L)
        plan = eph.NttPlan(q, lg)
        per_poly = L * N * 8
        batch = max(1, int(a.bytes * (1 << 30) // per_poly))
        x = torch.randint(0, 1 << 62, (batch, L, N), dtype=torch.int64, device=dev)
        qt = torch.tensor([int(v) for v in q], dtype=torch.int64, device=dev).view(1, L, 1)
        x = torch.remainder(x, qt)
        res = {}
        for name, fn in (("ntt_fwd", eph.ntt_fwd), ("ntt_inv", eph.ntt_inv)):
            for _ in range(3):
                fn(plan, x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                fn(plan, x)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            gbs = 2 * batch * per_poly / (ms / 1e3) / 1e9
            res[name] = {"ms": round(ms, 4), "GB_s": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4),
                         "butterflies_G_s": round(batch * L * (N // 2) * lg / (ms / 1e3) / 1e9, 1)}
        # MAC: D terms of ct [D][L][2][N] and pt [D][L][N]
        D = max(1, int(a.bytes * (1 << 30) // (3 * per_poly)))
        ct = torch.remainder(torch.randint(0, 1 << 62, (D, L, 2, N), dtype=torch.int64, device=dev), qt.view(1, L, 1, 1))
        pt = torch.remainder(torch.randint(0, 1 << 62, (D, L, N), dtype=torch.int64, device=dev), qt)
        out = torch.empty((L, 2, N), dtype=torch.int64, device=dev)
        for _ in range(3):
            eph.mac(plan, ct, pt, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            eph.mac(plan, ct, pt, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        gbs = 3 * D * per_poly / (ms / 1e3) / 1e9
        res["mac"] = {"D": D, "ms": round(ms, 4), "GB_s": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4)}
        print(json.dumps({"workload": "c5", "log2N": lg, "L": L, "bits": bits, "batch": batch,
                          "hbm_peak_gbs": hbm, **res}), flush=True)
        del x, ct, pt, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
