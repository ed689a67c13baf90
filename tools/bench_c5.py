#!/usr/bin/env python
"""c5 kernel microbench (BASELINE.json configs[4]): standalone negacyclic NTT (forward,
inverse) and the pointwise ct x pt MAC on uniform residues, one JSON line per
(N, L, prime class, word, batch) point -- the points of ephdc_inputs.c5_points, each
one parity-checked by tests/test_gpu_c5_sweep.py on the same seeded device inputs.

GB/s = algorithmic bytes / CUDA-event time on the launching stream (warm-up first):
  NTT: read + write of batch x L x N words (in place);
  MAC: read of D x L x (2 + 1) x N words (two ciphertext residues + one plaintext).
Small batches are latency-bound by construction (one polynomial per prime cannot fill
148 SMs); working sets above 1 GiB stream from HBM (L2 = 126 MB).  Every line carries
the nvidia-smi clock record of its timed region (bench.ClockSampler).
Peak: MEASURED_PEAKS.json hbm_gbs.

usage: python tools/bench_c5.py [--points quick|all] [--reps 5] [--only 13:9:48:8]
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
    ap.add_argument("--points", default="quick", choices=["quick", "all"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="", help="lg:L:bits:wordbytes[,...]")
    ap.add_argument("--max-batch-only", action="store_true", help="time only the largest batch of each point")
    ap.add_argument("--alt-teams", action="store_true", help="A/B: the other warp layout of the c5 kernels at N = 2^13")
    ap.add_argument("--u32-generic", action="store_true", help="A/B: the general u32 kernels instead of ntt32_c5.cu")
    a = ap.parse_args()
    import torch
    import ephdc_inputs as inp
    import paper_2511_00737_b200 as eph
    from bench import ClockSampler, measured_peaks

    hbm = measured_peaks().get("hbm_gbs", 6552.0)
    only = {tuple(int(v) for v in s.split(":")) for s in a.only.split(",") if s}
    dev = torch.device("cuda", 0)

    def timed(fn, reps):
        # >= 2 warm-ups; the timed region lasts >= 0.6 s so the clock sampler sees it
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        one = max(e0.elapsed_time(e1), 1e-3)
        reps = max(reps, int(600.0 / one) + 1)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    for lg, L, bits, wb, batches in inp.c5_points(a.points):
        if only and (lg, L, bits, wb) not in only:
            continue
        N = 1 << lg
        q = eph.find_ntt_primes(lg, [bits] * L)
        plan = eph.NttPlan(q, lg, alt_teams=a.alt_teams, u32_generic=a.u32_generic)
        if wb == 4 and not plan.u32_words:
            continue
        fwd, inv, mac = (eph.ntt_fwd, eph.ntt_inv, eph.mac) if wb == 8 else (eph.ntt_fwd32, eph.ntt_inv32, eph.mac32)
        dt = torch.int64 if wb == 8 else torch.int32
        seed = lg * 1000 + L * 10 + bits + wb
        base = inp.c5_residues_torch(q, max(batches), N, seed, dev, dt)
        per_poly = L * N * wb
        for batch in (batches[-1:] if a.max_batch_only else batches):
            x = base[:batch]
            reps = a.reps
            clk = ClockSampler(0)
            clk.start()
            res = {}
            for name, fn in (("ntt_fwd", fwd), ("ntt_inv", inv)):
                ms = timed(lambda: fn(plan, x), reps)
                gbs = 2 * batch * per_poly / (ms / 1e3) / 1e9
                res[name] = {"ms": round(ms, 5), "GB_s": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4),
                             "butterflies_G_s": round(batch * L * (N // 2) * lg / (ms / 1e3) / 1e9, 1)}
            res["clocks"] = clk.stop()
            res["kernels"] = {"fwd": plan.fwd_kernel if wb == 8 else plan.u32_kernel,
                              "inv": plan.inv_kernel if wb == 8 else plan.u32_kernel}
            print(json.dumps({"workload": "c5", "log2N": lg, "alt_teams": a.alt_teams, "L": L, "bits": bits, "word_bits": 8 * wb,
                              "batch": batch, "bytes_per_launch": 2 * batch * per_poly, "hbm_peak_gbs": hbm,
                              **res}), flush=True)
        del base
        torch.cuda.empty_cache()
        # MAC: D terms of ct [D][L][2][N] and pt [D][L][N] (~2 GiB)
        D = max(1, min(inp.c5_max_batch(lg, L, wb), (2 << 30) // (3 * per_poly)))
        mods = [q[j] for j in range(L) for _ in range(2)]
        ct = inp.c5_residues_torch(mods, D, N, seed + 1, dev, dt).view(D, L, 2, N)
        pt = inp.c5_residues_torch(q, D, N, seed + 2, dev, dt)
        out = torch.empty((L, 2, N), dtype=dt, device=dev)
        clk = ClockSampler(0)
        clk.start()
        ms = timed(lambda: mac(plan, ct, pt, out), a.reps)
        c = clk.stop()
        gbs = 3 * D * per_poly / (ms / 1e3) / 1e9
        print(json.dumps({"workload": "c5", "op": "mac", "log2N": lg, "L": L, "bits": bits, "word_bits": 8 * wb,
                          "D": D, "ms": round(ms, 4), "GB_s": round(gbs, 1), "frac_hbm": round(gbs / hbm, 4),
                          "hbm_peak_gbs": hbm, "clocks": c}), flush=True)
        del ct, pt, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
