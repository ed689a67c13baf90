"""findDmax (Algorithm 1) on the GPU (-m gpu).

tools/find_dmax.py evaluates 1000 random ct x pt dot products per (N, log2 t) as the
batches of ONE ephdc_infer_batch_prefix call and bisects, per trial, between a length
that decrypts correctly and one that does not.  Checked here on small trial counts:
  * ephdc_infer_batch_prefix = the oracle's evaluation over the same dim prefixes
    (bit-exact ciphertexts), so every probed D is a real evaluation;
  * the found D_i decrypts correctly and D_i + 1 does not -- decided by the ORACLE's
    Python-integer decryption compared with brute-force dot products mod t;
  * D_max(N, T-1) >= D_max(N, T) (the monotone trade-off of
    Fig. "D_max for various N and log2 t").
"""
import dataclasses
import os
import sys

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle.bfv import OracleBFV

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import find_dmax as fd  # noqa: E402

LOGN, T_HI = 11, 16      # N = 2^11, q = 2 x 27 bits (54); predicted D_max ~ 10^1 at T = 16


def _oracle_for(p, D):
    cfg = dataclasses.replace(inp.CONFIGS["c1"], name="dmax", log2N=LOGN, t_bits=p.t.bit_length(), t_fixed=p.t,
                              q_bits=fd.Q_BITS[LOGN], k=p.k, D_live=D, D_stored=D, Cbits=4)   # q: the SPEC cap, 54 bits
    o = OracleBFV(cfg)
    assert o.t == p.t and o.q == p.q
    o.keygen(1000)
    return o


def _oracle_correct(p, o, model, b, D):
    """Oracle evaluation of trial b over its first D dims, decrypted with Python integers."""
    H = p.H[:D, b * p.B:(b + 1) * p.B].cpu().numpy()
    o.D_live = D
    ct = o.infer_batch(H, p.B, 0, model=np.ascontiguousarray(model[:D]))
    slots = o.decrypt(ct)
    S = (H.astype(np.int64).T @ p.C[:, :D].astype(np.int64).T).reshape(-1)
    want = S % p.t
    return bool(np.array_equal(np.asarray(slots[: p.B * p.k], dtype=np.int64) % p.t, want)), ct


def test_find_dmax_literal_small():
    p = fd.Probe(LOGN, T_HI, trials=6, dcap=128)
    Di, cens, evals = p.find_dmax()
    assert evals >= 2
    o = _oracle_for(p, 128)
    model = o.encrypt_dims(p.C, 2000, 0, 128)
    # the prefix evaluation is the oracle's evaluation, bit for bit
    dims = np.array([min(int(d) + 1, 128) for d in Di], dtype=np.uint32)
    got = p.eph.infer_batch_prefix(p.ctx, p.model, p.ws, p.H, p.nq, dims).cpu().numpy().view(np.uint64)
    for b in range(2):
        ok, ct = _oracle_correct(p, o, model, b, int(dims[b]))
        assert np.array_equal(got[b], ct), b
    for b in range(p.trials):
        if Di[b] > 0:
            assert _oracle_correct(p, o, model, b, int(Di[b]))[0], (b, Di[b])
        if not cens[b]:
            assert not _oracle_correct(p, o, model, b, int(Di[b]) + 1)[0], (b, Di[b])


def test_find_dmax_monotone_in_log2t():
    means = []
    for T in (T_HI + 1, T_HI, T_HI - 1):   # t = 114689, 61441, 12289 (no 15-bit prime = 1 mod 4096)
        p = fd.Probe(LOGN, T, trials=16, dcap=4096)
        Di, _, _ = p.find_dmax()
        means.append(float(Di.mean()))
        del p
        torch.cuda.empty_cache()
    assert means[0] <= means[1] <= means[2], means
