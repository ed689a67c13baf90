#!/usr/bin/env python
"""Fused-kernel time and (under ncu) DRAM traffic at c4 for grid-order / chunk-size
variants, all in one process so that one ncu invocation covers every variant.

Variant = (EPHDC_F64_FLAGS, EPHDC_F64_BG, EPHDC_F64_G); BG / G = 0 keep the planner's
choice (f64_grid).  profiles/r01/l2sched/sweep*.txt were taken when flags bit 4 selected
the batch-fastest block order that is now the only order.  Without --ncu: one warm-up step and
`--reps` timed steps per variant (CUDA events around the fused launch), one JSON line
each.  With --ncu: exactly one step per variant (profile with -k regex:k_ntt_mac_f64
-c <n variants>), launches in the order printed.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DEFAULT = ["0,0,0", "0,8,0", "0,29,0", "0,0,100", "0,0,589"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--variants", nargs="+", default=DEFAULT)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--ncu", action="store_true")
    a = ap.parse_args()
    import torch
    import ephdc_inputs as inp
    import paper_2511_00737_b200 as eph
    from paper_2511_00737_b200 import pipeline as ppipe

    cfg = inp.CONFIGS[a.config]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr)
    ctx, model, nq = ps.ctx, ps.model, cfg.nq
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    ws = eph.Workspace(ctx, nq)
    H = torch.empty((cfg.D_live, nq), dtype=torch.int8, device="cuda")
    out = torch.empty(ctx.ct_shape(nq), dtype=torch.int64, device="cuda")
    eph.encode_queries(ctx, X, ps.P_dev, H)
    ref = None
    for v in a.variants:
        f, bg, g = v.split(",")
        os.environ["EPHDC_F64_FLAGS"] = f
        if bg != "0":
            os.environ["EPHDC_F64_BG"] = bg
        else:
            os.environ.pop("EPHDC_F64_BG", None)
        if g != "0":
            os.environ["EPHDC_F64_G"] = g
        else:
            os.environ.pop("EPHDC_F64_G", None)
        if a.ncu:
            eph.infer_batch(ctx, model, ws, H, nq, out)
            torch.cuda.synchronize()
            print(json.dumps({"variant": v}), flush=True)
            continue
        eph.infer_batch(ctx, model, ws, H, nq, out)
        torch.cuda.synchronize()
        got = out.cpu()
        if ref is None:
            ref = got
        same = bool(torch.equal(got, ref))
        ws.set_timing(True)
        ws.timing()
        for _ in range(a.reps):
            eph.infer_batch(ctx, model, ws, H, nq, out)
        torch.cuda.synchronize()
        kt = ws.timing()
        ws.set_timing(False)
        print(json.dumps({"variant": v, "ntt_mac_ms": round(kt["ntt_mac"][0] / a.reps, 3),
                          "same_output": same}), flush=True)


if __name__ == "__main__":
    main()
