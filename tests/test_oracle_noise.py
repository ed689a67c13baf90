"""Noise budget of the client evaluation (PAPER.md l.476-484 findDmax's question, answered
by measurement and a closed form; not gpu).

Algorithm 1's findDmax searches, by repeated decryption, the largest D whose
ct-pt dot product still decrypts.  The noise of sum_d CT_d * PT_d grows like a random
walk: its infinity norm is ~ r_t(Q) sqrt(N) (t/6) sqrt(D) (r_t(Q) = Q mod t, the wrap
term of Delta * t = Q - r_t(Q); plaintext coefficients uniform mod t), so

    D_max ~ D * (Delta/2 / noise(D))^2 .

This test measures the noise of the oracle's scores ciphertexts at c1q3 and c2 for
several D, checks it against the closed form (within 3 bits) and that it stays below
Delta/2 (decryption correct), and prints the extrapolated D_max (reading #21
discusses why the literal per-D search is not run: at c2-c4 D_max exceeds any D by
many orders of magnitude, and c1 literal has D_max = 0).
"""
import math

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import hdc, pipeline


@pytest.mark.parametrize("name,Ds", [("c1q3", [1, 16, 256, 1024]), ("c2", [4, 64, 1024])])
def test_noise_growth_matches_closed_form(name, Ds):
    cfg = inp.CONFIGS[name]
    nq = 16
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    m = pipeline.build_model(cfg, P, Xtr, ytr)
    bfv = m.bfv
    H = pipeline.encode_queries(m, P, Xq)
    r = bfv.Q % bfv.t
    half_delta_bits = math.log2(bfv.delta_big / 2)
    out = []
    for D in Ds:
        bfv.D_live = D                  # class_hv rows must then have stride D
        ct = bfv.infer_batch(H, nq, 0, class_hv=np.ascontiguousarray(m.class_hv[:, :D]), enc_seed=m.enc_seed)
        S = hdc.scores(H[:D], m.class_hv[:, :D])
        slots = np.zeros(bfv.N, dtype=np.int64)
        slots[: bfv.k * nq] = S.reshape(-1)
        bits = bfv.noise_bits(ct, slots)
        pred = math.log2(r * math.sqrt(bfv.N) * bfv.t / 6 * math.sqrt(D)) + 1.5
        dmax = D * 2 ** (2 * (half_delta_bits - bits))
        out.append((D, round(bits, 2), round(pred, 2), f"{dmax:.3g}"))
        assert abs(bits - pred) < 3.0, (name, D, bits, pred)
        assert bits < half_delta_bits
    bfv.D_live = cfg.D_live
    print(name, "Delta/2 = 2^%.1f" % half_delta_bits, "(D, noise bits, closed form, D_max estimate):", out)
