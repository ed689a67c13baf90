"""Pins of the oracle's BFV pipeline (not gpu).

* Dec(Enc(m)) = m and Dec(Enc(m) * p) = m (.) p mod t (north_star);
* decrypted scores equal brute-force integer dot products, labels the brute-force
  argmax (north_star);
* op budget D MulCP, D-1 AddCC, 0 rotations (golden/paper_values.json);
* batch size floor(N/k) against the paper's printed batch sizes;
* c1 literal is noise-infeasible: decryption after one product is wrong.
"""
import json
import os

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import core, hdc, pipeline
from oracle.bfv import OracleBFV

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _setup(name, nq=None):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, yq = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    m = pipeline.build_model(cfg, P, Xtr, ytr)
    return cfg, m, P, Xq, yq


def _tile(m, d):
    bfv = m.bfv
    v = np.zeros(bfv.N, dtype=np.int64)
    i = np.arange(bfv.k * bfv.B)
    v[: bfv.k * bfv.B] = m.class_hv[i % bfv.k, d]
    return v % bfv.t


def _pt_hat(bfv, w):
    """p_hat_j = NTT_j(centered lift of encode(w)) written out independently of or_plaintext_ntts."""
    msg = bfv.slot_encode(np.asarray(w, dtype=np.uint64))
    out = []
    for j, q in enumerate(bfv.q):
        lifted = np.array([int(x) if int(x) <= (bfv.t - 1) // 2 else int(x) - bfv.t + q for x in msg],
                          dtype=np.uint64)
        out.append(core.ntt_fwd(lifted, bfv.logN, q, bfv.psi[j]))
    return out


def test_paper_batch_sizes():
    gold = json.load(open(os.path.join(GOLD, "paper_values.json")))
    for row in gold["batch_sizes"]:
        assert row["N"] // row["k"] == row["B"]
    for name, B in (("c1", 512), ("c2", 2048), ("c3", 819), ("c4", 2340)):
        assert OracleBFV(inp.CONFIGS[name]).B == B


def test_keygen_deterministic():
    b1 = OracleBFV(inp.CONFIGS["c1q3"])
    b2 = OracleBFV(inp.CONFIGS["c1q3"])
    assert np.array_equal(b1.keygen(5), b2.keygen(5))
    assert not np.array_equal(b1.keygen(5), b2.keygen(6))


@pytest.mark.parametrize("name", ["c1q3", "c2"])
def test_enc_dec_roundtrip_and_ct_pt_product(name):
    cfg, m, *_ = _setup(name, nq=16)
    bfv = m.bfv
    for d in (0, 1, cfg.D_live - 1):
        ct = m.bfv.encrypt_dims(m.class_hv, m.enc_seed, d, 1)[0]          # [L][2][N]
        ctk = np.ascontiguousarray(ct.transpose(1, 0, 2))                  # [2][L][N]
        assert np.array_equal(bfv.decrypt(ctk), _tile(m, d))              # Dec(Enc(m)) = m
        w = np.random.default_rng(d).integers(0, bfv.t, size=bfv.N, dtype=np.uint64)
        ph = _pt_hat(bfv, w)
        prod = np.empty_like(ctk)
        for c in range(2):
            for j, q in enumerate(bfv.q):
                prod[c, j] = np.array((ctk[c, j].astype(object) * ph[j].astype(object)) % q, dtype=np.uint64)
        want = (_tile(m, d).astype(object) * w.astype(object)) % bfv.t
        assert np.array_equal(bfv.decrypt(prod), np.array(want, dtype=np.uint64))   # Dec(Enc(m)*p) = m.p
        assert bfv.noise_bits(prod, want) < np.log2(float(bfv.delta_big)) - 1


def test_c1_literal_is_noise_infeasible():
    cfg, m, *_ = _setup("c1", nq=16)
    bfv = m.bfv
    ct = np.ascontiguousarray(bfv.encrypt_dims(m.class_hv, m.enc_seed, 0, 1)[0].transpose(1, 0, 2))
    # even a fresh ciphertext fails: r_t(q)*m/q reaches (q mod t)*(t-1)/q ~ 0.87 > 1/2 at one 30-bit q
    assert (bfv.decrypt(ct) == _tile(m, 0)).mean() < 0.9
    w = np.random.default_rng(0).integers(0, bfv.t, size=bfv.N, dtype=np.uint64)
    ph = _pt_hat(bfv, w)
    q = bfv.q[0]
    prod = np.stack([np.array((ct[c, 0].astype(object) * ph[0].astype(object)) % q, dtype=np.uint64)
                     for c in range(2)])[:, None, :]
    want = np.array((_tile(m, 0).astype(object) * w.astype(object)) % bfv.t, dtype=np.uint64)
    got = bfv.decrypt(prod)
    assert (got == want).mean() < 0.01                       # noise wraps


@pytest.mark.parametrize("name,nq", [("c1q3", 16), ("c1q3", 700), ("c2", 300)])
def test_scores_equal_bruteforce(name, nq):
    cfg, m, P, Xq, yq = _setup(name, nq=nq)
    H = pipeline.encode_queries(m, P, Xq)
    cts = pipeline.infer_all(m, H)
    S, lab = m.bfv.decode_scores(cts, nq)
    Sref = hdc.scores(H, m.class_hv)
    assert np.array_equal(S, Sref)
    assert np.array_equal(lab, hdc.argmax_lowest(Sref))
    assert (lab == yq).mean() > 0.9                           # the synthetic clusters separate


def test_op_budget_counters():
    cfg, m, P, Xq, _ = _setup("c1q3", nq=16)
    H = pipeline.encode_queries(m, P, Xq)
    cnt = np.zeros(3, dtype=np.uint64)
    m.bfv.infer_batch(H, 16, 0, class_hv=m.class_hv, enc_seed=m.enc_seed, counters=cnt)
    D = cfg.D_live
    assert cnt.tolist() == [D, D - 1, 0]


def test_stored_model_equals_on_the_fly():
    cfg, m, P, Xq, _ = _setup("c1q3", nq=16)
    H = pipeline.encode_queries(m, P, Xq)
    model = m.bfv.encrypt_dims(m.class_hv, m.enc_seed, 0, cfg.D_live)
    a = m.bfv.infer_batch(H, 16, 0, model=model)
    b = m.bfv.infer_batch(H, 16, 0, class_hv=m.class_hv, enc_seed=m.enc_seed)
    assert np.array_equal(a, b)


def test_plaintext_ntts_match_independent_writeout():
    cfg, m, P, Xq, _ = _setup("c1q3", nq=600)
    H = pipeline.encode_queries(m, P, Xq)
    bfv = m.bfv
    for b in (0, 1):
        got = bfv.plaintext_ntts(H, 600, b, 5, 2)
        for dd in range(2):
            d = 5 + dd
            nb = min(bfv.B, 600 - b * bfv.B)
            w = np.zeros(bfv.N, dtype=np.int64)
            w[: bfv.k * nb] = np.repeat(H[d, b * bfv.B: b * bfv.B + nb].astype(np.int64), bfv.k)
            ph = _pt_hat(bfv, w % bfv.t)
            for j in range(bfv.L):
                assert np.array_equal(got[dd, j], ph[j])
