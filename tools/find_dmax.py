#!/usr/bin/env python
"""findDmax on the GPU (Algorithm 1 lines 17-24).

Algorithm 1 repeats, 1000 times, "grow D while evalHEcomputation(N, T, D+1) decrypts
correctly" and returns the mean D_i.  Each trial here is one scores ciphertext of the
real hot path (encode + pack + lift/NTT/MAC over D dims, `ephdc_infer_batch`) on
synthetic queries; `ephdc_noise_probe` measures its noise exactly on the GPU.  Instead
of re-evaluating every D (at c2-c4 the budget allows ~1e20+ dims, so the literal loop
would not terminate -- DESIGN.md reading #21), D_i is extrapolated from the measured
noise with the random-walk growth |e| ~ sqrt(D) that tests/test_oracle_noise.py pins
against the closed form:  D_i = D * (Delta/2 / |e_i|)^2  (D_i = 0 when trial i already
fails at D; that is the literal outcome at c1).  --dims evaluates several D (the
model's first D dims) and checks the sqrt(D) growth on the GPU as well.

usage: python tools/find_dmax.py [--configs c1 c1q3 c2 c3 c4] [--trials 1000] [--dims ...]
One JSON line per (config, D).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c1", "c1q3", "c2", "c3", "c4"])
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--dims", nargs="*", type=int, default=[], help="D values (default: the config's D_live)")
    a = ap.parse_args()
    import torch
    import ephdc_inputs as inp
    import paper_2511_00737_b200 as eph
    from paper_2511_00737_b200 import pipeline as ppipe

    for name in a.configs:
        base = inp.CONFIGS[name]
        for D in (a.dims or [base.D_live]):
            if D > base.D_live:
                continue
            cfg = dataclasses.replace(base, D_live=D)
            t, q = ppipe.primes_for(cfg)
            Q = math.prod(int(x) for x in q)
            half_delta = (Q // t) // 2
            Xtr, ytr, _, _ = inp.gen_features(cfg, 1)
            P = inp.gen_projection(cfg)
            ps = ppipe.build(cfg, P, Xtr, ytr)
            B = ps.ctx.B
            nq = a.trials * B
            rng = np.random.default_rng([cfg.seed, 77, D])
            hi = 256 if cfg.feat_unsigned else 128
            Xq = rng.integers(0 if cfg.feat_unsigned else -128, hi, size=(nq, cfg.F),
                              dtype=np.uint8 if cfg.feat_unsigned else np.int8)
            X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
            ws = eph.Workspace(ps.ctx, nq)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            H = eph.encode_queries(ps.ctx, X, ps.P_dev)
            cts = eph.infer_batch(ps.ctx, ps.model, ws, H, nq)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            bits, flags, lg = eph.noise_probe(ps.ctx, ps.sk, cts)
            t2 = time.perf_counter()
            hd = math.log2(half_delta)
            fails = (lg >= hd) | (flags != 0)
            Di = np.where(fails, 0.0, D * np.exp2(2.0 * (hd - lg)))
            line = {"workload": name, "D": D, "trials": int(a.trials), "N": ps.ctx.N, "L": ps.ctx.L, "t": int(t),
                    "log2_half_delta": round(hd, 3),
                    "noise_log2_mean": round(float(lg.mean()), 3), "noise_log2_max": round(float(lg.max()), 3),
                    "noise_bits_max": int(bits.max()), "decrypt_fail_trials": int(fails.sum()),
                    "D_max_mean": float(Di.mean()), "D_max_min": float(Di.min()),
                    "closed_form_noise_log2": round(math.log2((Q % t) * math.sqrt(ps.ctx.N) * t / 6 * math.sqrt(D)) + 1.5, 3),
                    "gpu_eval_s": round(t1 - t0, 3), "gpu_probe_s": round(t2 - t1, 3)}
            print(json.dumps(line), flush=True)
            del cts, H, X, ws, ps
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
