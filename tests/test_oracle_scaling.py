"""Pins of the oracle's accumulator scaling (SPEC S:399-402,
S:430) -- NEXT #1 of SURVEY 8(f) (not gpu).

* the modular-inverse arithmetic of SPEC's worked example (t = 17, s = 2: 10 * 9 = 5,
  11 * 9 = 14 mod 17), on a real ciphertext: scale a fresh encryption and decrypt;
* an all-ones schedule is the identity: bit-identical ciphertexts to the
  unscaled evaluation, for any g (including a ragged last group);
* a non-trivial schedule decrypts to the closed form
      sum_J (sum_{d in J} h[d] C[d]) * prod_{J' >= J} s_J'^-1  (mod t)
  computed with Python integers from H and the class HVs (independent of the BFV code);
* op budget: D MulCP, D - 1 AddCC, ceil(D/g) scaling multiplies, 0 rotations.
"""
import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import hdc, pipeline


def _setup(name, nq):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    m = pipeline.build_model(cfg, P, Xtr, ytr)
    H = pipeline.encode_queries(m, P, Xq)
    return cfg, m, H


def test_spec_worked_example_mod_17():
    # S:462 (t = 17, s = 2, s^-1 = 9): 10 -> 5 exactly, 11 -> 14 (wraps)
    assert pow(2, -1, 17) == 9
    assert (10 * 9) % 17 == 5 and (11 * 9) % 17 == 14


@pytest.mark.parametrize("g", [512, 100])
def test_all_ones_schedule_is_identity(g):
    cfg, m, H = _setup("c1q3", 16)
    ng = -(-cfg.D_live // g)
    cnt = {}
    got = m.bfv.infer_batch_scaled(H, 16, 0, g, [1] * ng, class_hv=m.class_hv, enc_seed=m.enc_seed, counters=cnt)
    want = m.bfv.infer_batch(H, 16, 0, class_hv=m.class_hv, enc_seed=m.enc_seed)
    assert np.array_equal(got, want)
    D = cfg.D_live
    assert cnt == {"mul_cp": D, "add_cc": D - 1, "scale": ng, "rot": 0}


def _closed_form(H, C, t, g, scales, nq):
    D = H.shape[0]
    k = C.shape[0]
    out = np.zeros((nq, k), dtype=np.int64)
    for q in range(nq):
        for c in range(k):
            tot = 0
            for J, s in enumerate(scales):
                d0, d1 = J * g, min(D, (J + 1) * g)
                part = sum(int(H[d, q]) * int(C[c, d]) for d in range(d0, d1))
                f = 1
                for s2 in scales[J:]:
                    f = f * pow(int(s2), -1, t) % t
                tot = (tot + part * f) % t
            out[q, c] = tot if tot <= (t - 1) // 2 else tot - t
    return out


@pytest.mark.parametrize("g,scales", [(512, [256, 256]), (300, [4096, 16384, 256, 4096])])
def test_scaled_evaluation_decrypts_to_closed_form(g, scales):
    # c1q3: t = 65537 = 2^16 + 1, so 2^-k = -2^(16-k) (mod t): powers of two have small
    # centered inverses and keep the noise growth (x 2^(16-k) per scaling) inside the
    # 34-bit margin.  (A scale like 3 has |lift(3^-1)| ~ 2^14.4 -- SURVEY 0.8's caveat:
    # a few such scalings exhaust the budget, see test_bad_schedule_exhausts_noise.)
    nq = 8
    cfg, m, H = _setup("c1q3", nq)
    ct = m.bfv.infer_batch_scaled(H, nq, 0, g, scales, class_hv=m.class_hv, enc_seed=m.enc_seed)
    S, _ = m.bfv.decode_scores(ct[None], nq)
    assert np.array_equal(S, _closed_form(H, m.class_hv, m.bfv.t, g, scales, nq))
    # and it is not the unscaled result
    assert not np.array_equal(S, hdc.scores(H, m.class_hv))


def test_bad_schedule_exhausts_noise():
    # scales with large centered inverses multiply the noise past Delta/2: the literal
    # procedure then fails to decrypt (documented reading #21)
    nq = 8
    cfg, m, H = _setup("c1q3", nq)
    scales = [3, 5, 3, 5]
    ct = m.bfv.infer_batch_scaled(H, nq, 0, 300, scales, class_hv=m.class_hv, enc_seed=m.enc_seed)
    S, _ = m.bfv.decode_scores(ct[None], nq)
    assert not np.array_equal(S, _closed_form(H, m.class_hv, m.bfv.t, 300, scales, nq))
