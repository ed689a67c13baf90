"""Pins of the oracle's HE-HDC-SR baseline (NEXT #3; not gpu):
the client's query ciphertexts decrypt to the interleaved query slots, and the
server's evaluation with plaintext class tiles decrypts to the brute-force dot
products -- the same scores EP-HDC's client-side evaluation yields."""
import numpy as np

import ephdc_inputs as inp
from oracle import hdc, pipeline


def test_sr_roundtrip_and_scores():
    cfg = inp.CONFIGS["c1q3"]
    nq = 700
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    m = pipeline.build_model(cfg, P, Xtr, ytr)
    bfv = m.bfv
    H = pipeline.encode_queries(m, P, Xq)
    Sref = hdc.scores(H, m.class_hv)
    for b in range(bfv.n_batches(nq)):
        qct = bfv.sr_encrypt_queries(H, nq, b, enc_seed=4242)
        nb = min(bfv.B, nq - b * bfv.B)
        for d in (0, 517, cfg.D_live - 1):
            slots = bfv.decrypt(qct[d].transpose(1, 0, 2))          # [L][2][N] -> [2][L][N]
            want = np.zeros(bfv.N, dtype=np.int64)
            i = np.arange(bfv.k * nb)
            want[: bfv.k * nb] = H[d, b * bfv.B + i // bfv.k]
            assert np.array_equal(slots.astype(np.int64), want % bfv.t)
        res = bfv.sr_server_eval(m.class_hv, qct)
        v = bfv.decrypt(res).astype(np.int64)
        v = np.where(v > (bfv.t - 1) // 2, v - bfv.t, v)
        S = v[: bfv.k * nb].reshape(nb, bfv.k)
        assert np.array_equal(S, Sref[b * bfv.B: b * bfv.B + nb])
