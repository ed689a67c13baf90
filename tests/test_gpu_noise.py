"""GPU noise probe (findDmax's measurement; NEXT #2) vs the oracle
(-m gpu).

ephdc_noise_probe returns, per scores ciphertext, the exact bit length of
max_i |x_i - Delta m_i| (x = c0 + c1 s in coefficient form, m = the rounded
decryption).  Where the decryption is correct that is the ciphertext noise, which the
oracle computes with Python integers against the EXPECTED plaintext (bfv.noise_max):
the bit lengths must be equal and the flag clear.  At c1 literal (noise margin -26
bits) the oracle's noise exceeds Delta/2 -- the decryption fails -- and the
probe's distance to the nearest codeword sits just below Delta/2.
"""
import math

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import hdc, pipeline as opipe

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_00737_b200 as eph  # noqa: E402
from paper_2511_00737_b200 import pipeline as ppipe  # noqa: E402


def _setup(name, nq):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, deterministic=True)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    H = eph.encode_queries(ps.ctx, X, ps.P_dev)
    ws = eph.Workspace(ps.ctx, nq)
    cts = eph.infer_batch(ps.ctx, ps.model, ws, H, nq)
    torch.cuda.synchronize()
    om = opipe.build_model(cfg, P, Xtr, ytr)
    H_or = opipe.encode_queries(om, P, Xq)
    return cfg, ps, cts, om, hdc.scores(H_or, om.class_hv)


def _expected_slots(bfv, S, b):
    slots = np.zeros(bfv.N, dtype=np.int64)
    rows = S[b * bfv.B:(b + 1) * bfv.B]
    slots[: bfv.k * rows.shape[0]] = rows.reshape(-1)
    return slots


@pytest.mark.parametrize("name,nq", [("c1q3", 700), ("c2", 300), ("c3", 900)])
def test_probe_matches_oracle_noise(name, nq):
    cfg, ps, cts, om, S = _setup(name, nq)
    bits, flags, lg = eph.noise_probe(ps.ctx, ps.sk, cts)
    got = cts.cpu().numpy().view(np.uint64)
    half_delta = om.bfv.delta_big // 2
    batches = range(got.shape[0]) if name != "c3" else (0, got.shape[0] - 1)
    for b in batches:
        worst = om.bfv.noise_max(got[b], _expected_slots(om.bfv, S, b))
        assert worst < half_delta                       # the decryption is correct ...
        assert int(bits[b]) == worst.bit_length(), b    # ... so the probe sees the noise
        assert flags[b] == 0
        assert abs(lg[b] - math.log2(worst)) < 1e-9
    assert np.all(bits < half_delta.bit_length())


def test_probe_at_failing_literal_c1():
    cfg, ps, cts, om, S = _setup("c1", 16)
    bits, flags, lg = eph.noise_probe(ps.ctx, ps.sk, cts)
    got = cts.cpu().numpy().view(np.uint64)
    delta = om.bfv.delta_big
    worst = om.bfv.noise_max(got[0], _expected_slots(om.bfv, S, 0))
    assert worst > delta // 2                            # decryption fails (margin -26 bits)
    # the rounded decryption's residual x - Delta m, m = round(t x / Q), is at most
    # Q/(2t) + m (Q/t - Delta) < Q/(2t) + t: here (t ~ 4 Delta) up to ~1.5 Delta
    Q, t = om.bfv.Q, om.bfv.t
    assert delta.bit_length() - 3 <= int(bits[0]) <= (Q // (2 * t) + t).bit_length()


def test_probe_empty_and_errors():
    cfg = inp.CONFIGS["c1q3"]
    Xtr, ytr, _, _ = inp.gen_features(cfg, 4)
    ps = ppipe.build(cfg, inp.gen_projection(cfg), Xtr, ytr, deterministic=True)
    empty = torch.empty((0, 2, ps.ctx.L, ps.ctx.N), dtype=torch.int64, device="cuda")
    bits, flags, lg = eph.noise_probe(ps.ctx, ps.sk, empty)
    assert bits.size == 0
    other = ppipe.build(cfg, inp.gen_projection(cfg), Xtr, ytr, deterministic=True)
    ct = torch.zeros((1, 2, ps.ctx.L, ps.ctx.N), dtype=torch.int64, device="cuda")
    with pytest.raises(eph.EphdcError) as e:
        eph.noise_probe(ps.ctx, other.sk, ct)
    assert e.value.status == 2                           # EPHDC_ECONTEXT
    # the all-zero ciphertext decrypts to m = 0 with zero noise
    bits, flags, lg = eph.noise_probe(ps.ctx, ps.sk, ct)
    assert bits[0] == 0 and flags[0] == 0 and lg[0] == 0.0
