#!/usr/bin/env python
"""One small end-to-end run of the hot path, checked against the oracle's decryption:
c1q3 by default (N = 1024), every kernel of a call -- encoder, pack+INTT_t, fused
lift+NTT+MAC, finalize -- plus the noise probe.  --flags sets the ephdc_plan flag bits
of the fused kernel (4 = the windowed WL = 2 tail that c3/c4 use), so that variant runs
at a small size.  (Meant for compute-sanitizer; the tool is closed on this GPU pool, so
it serves as the small-case check against the oracle.  The library reads no
environment variables: variants go through the plan argument only.)

usage: python tools/sanitize_run.py [--config c1q3] [--nq 700] [--flags 4]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1q3")
    ap.add_argument("--nq", type=int, default=700)
    ap.add_argument("--flags", type=lambda v: int(v, 0), default=0, help="ephdc_plan flag bits (tests / A/B only)")
    a = ap.parse_args()
    import torch
    import ephdc_inputs as inp
    import paper_2511_00737_b200 as eph
    from paper_2511_00737_b200 import pipeline as ppipe
    from oracle import hdc, pipeline as opipe

    cfg = inp.CONFIGS[a.config]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, a.nq)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    H = eph.encode_queries(ps.ctx, X, ps.P_dev)
    ws = eph.Workspace(ps.ctx, a.nq, plan={"flags": a.flags} if a.flags else None)
    cts = eph.infer_batch(ps.ctx, ps.model, ws, H, a.nq)
    bits, flags, _ = eph.noise_probe(ps.ctx, ps.sk, cts)
    torch.cuda.synchronize()
    S, lab = eph.decrypt_scores(ps.ctx, ps.sk, cts.cpu().numpy().view(np.uint64), a.nq)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    Sref = hdc.scores(opipe.encode_queries(om, P, Xq), om.class_hv)
    ok = np.array_equal(S, Sref) and not flags.any()
    print(f"sanitize_run {a.config} nq={a.nq} plan_flags={a.flags} "
          f"scores {'ok' if ok else 'MISMATCH'} noise_bits={bits.tolist()}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
