#!/usr/bin/env python
"""Client-side (EP-HDC) vs server-side (HE-HDC-SR) HE on one B200, per batch of B
queries -- the B200 version of PAPER.md Table "Message size and client runtime"
(l.763-786: 9.1x client runtime, D x message size).  One JSON line per config.

EP-HDC client  = encode_queries + infer_batch (pack+INTT_t, lift+NTT_q+MAC) for B queries
HE-HDC-SR client = encode_queries + sr_encrypt_queries (D ciphertexts) for B queries
HE-HDC-SR server = sr_evaluate (D MulCP with plaintext class tiles)
Messages: EP-HDC sends one scores ciphertext (bit-packed, ephdc_scores_message_bytes);
HE-HDC-SR uploads D ciphertexts (same packing) and receives one.
CUDA-event times, warm-up 3, median of >= 5 repetitions spanning >= 0.6 s, each
measurement with the nvidia-smi clock record of its timed region (bench.ClockSampler).

usage: python tools/bench_sr.py [--configs c2 c3 c4]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=5, warm=3):
    """(median ms, clock record): >= reps repetitions and >= 0.6 s under the sampler."""
    import torch
    from bench import ClockSampler
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    clk = ClockSampler(0)
    clk.start()
    ts = []
    while len(ts) < reps or sum(ts) < 600.0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), clk.stop()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2", "c3", "c4"])
    a = ap.parse_args()
    import torch
    import ephdc_inputs as inp
    import paper_2511_00737_b200 as eph
    from paper_2511_00737_b200 import pipeline as ppipe

    for name in a.configs:
        cfg = inp.CONFIGS[name]
        Xtr, ytr, Xq, _ = inp.gen_features(cfg)
        P = inp.gen_projection(cfg)
        ps = ppipe.build(cfg, P, Xtr, ytr)
        ctx = ps.ctx
        nq = min(cfg.nq, ctx.B)                       # one full batch of B queries
        X = torch.from_numpy(np.ascontiguousarray(Xq[:nq]).view(np.int8)).cuda()
        ws = eph.Workspace(ctx, nq)
        H = torch.empty((cfg.D_live, nq), dtype=torch.int8, device="cuda")
        out = torch.empty(ctx.ct_shape(nq), dtype=torch.int64, device="cuda")
        qct = torch.empty((cfg.D_live, ctx.L, 2, ctx.N), dtype=torch.int64, device="cuda")
        pt = eph.sr_model_plaintexts(ctx, ps.class_hv)
        res = torch.empty((2, ctx.L, ctx.N), dtype=torch.int64, device="cuda")

        def ep_client():
            eph.encode_queries(ctx, X, ps.P_dev, H)
            eph.infer_batch(ctx, ps.model, ws, H, nq, out)

        def sr_client():
            eph.encode_queries(ctx, X, ps.P_dev, H)
            eph.sr_encrypt_queries(ctx, ps.sk, ws, H, nq, 0, None, qct)

        def sr_server():
            eph.sr_evaluate(ctx, pt, qct, res)

        (t_ep, c_ep), (t_src, c_src), (t_srs, c_srs) = timed(ep_client), timed(sr_client), timed(sr_server)
        msg1 = eph.scores_message_bytes(ctx, 1)
        line = {"workload": name, "queries_per_batch": nq, "N": ctx.N, "L": ctx.L, "D": cfg.D_live,
                "ep_hdc_client_ms": round(t_ep, 3), "he_hdc_sr_client_ms": round(t_src, 3),
                "he_hdc_sr_server_ms": round(t_srs, 3), "client_ratio_sr_over_ep": round(t_src / t_ep, 2),
                "ep_hdc_upload_bytes": msg1, "he_hdc_sr_upload_bytes": msg1 * cfg.D_live,
                "message_ratio": cfg.D_live,
                "clocks": {"ep_hdc_client": c_ep, "he_hdc_sr_client": c_src, "he_hdc_sr_server": c_srs},
                "paper": "P:778-786 (Ryzen 3970X, 1 core, Pyfhel): SR client 351.95 ms vs EP 43.99 ms at N=2^11 D=1K"}
        print(json.dumps(line), flush=True)
        del qct, pt, out, H, X, ws, ps
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
