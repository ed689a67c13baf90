"""Full-size parity in the launch configuration bench.py times (-m gpu).

BASELINE.json configs[2] (c3, 8192 queries = 11 batches) and configs[3] (c4, 65536
queries = 29 batches, N = 16384, 9 x 48-bit primes): the whole step runs through the
same calls bench.py times (encode_queries + infer_batch over every batch, one fused
launch).  Checked against the oracle:
  * H (all queries) bit-exact;
  * the scores ciphertexts of EVERY batch bit-exact against the oracle's evaluation
    (the oracle encrypts its model once per test and evaluates batch by batch);
  * every batch decrypts to the brute-force integer dot products, every label is the
    lowest-index argmax.
The integer-pipe kernel (ephdc_params.arith = INT, the path AUTO takes for primes >=
2^50) runs the same full-size step and must give the same ciphertexts.
"""
import dataclasses

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import hdc, pipeline as opipe

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_00737_b200 as eph  # noqa: E402
from paper_2511_00737_b200 import pipeline as ppipe  # noqa: E402


def _run_step(ps, cfg, Xq, nq):
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    ws = eph.Workspace(ps.ctx, nq)
    H = torch.empty((cfg.D_live, nq), dtype=torch.int8, device="cuda")
    out = torch.empty(ps.ctx.ct_shape(nq), dtype=torch.int64, device="cuda")
    eph.encode_queries(ps.ctx, X, ps.P_dev, H)
    eph.infer_batch(ps.ctx, ps.model, ws, H, nq, out)
    torch.cuda.synchronize()
    return H.cpu().numpy(), out.cpu().numpy().view(np.uint64).copy()


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_fullsize_step_parity(name):
    cfg = inp.CONFIGS[name]
    nq = cfg.nq
    Xtr, ytr, Xq, _ = inp.gen_features(cfg)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, deterministic=True)
    assert ps.ctx.arith == "f64"
    H, got = _run_step(ps, cfg, Xq, nq)
    nb = got.shape[0]

    om = opipe.build_model(cfg, P, Xtr, ytr)
    assert np.array_equal(ps.class_hv, om.class_hv)
    H_or = opipe.encode_queries(om, P, Xq)
    assert np.array_equal(H, H_or)
    model = om.bfv.encrypt_dims(om.class_hv, om.enc_seed, 0, cfg.D_live)
    for b in range(nb):
        want = om.bfv.infer_batch(H_or, nq, b, model=model)
        assert np.array_equal(got[b], want), f"batch {b}"
    del model

    S, lab = eph.decrypt_scores(ps.ctx, ps.sk, got, nq)
    Sref = hdc.scores(H_or, om.class_hv)
    assert np.array_equal(S, Sref)
    assert np.array_equal(lab.astype(np.int64), hdc.argmax_lowest(Sref))

    # the integer-pipe fused kernel on the same full-size step
    del ps
    torch.cuda.empty_cache()
    ps_int = ppipe.build(cfg, P, Xtr, ytr, arith=1, deterministic=True)
    assert ps_int.ctx.arith == "int"
    _, got_int = _run_step(ps_int, cfg, Xq, nq)
    assert np.array_equal(got_int, got)


def test_int_path_large_primes_n16384():
    """N = 2^14 with nine primes of ~55 bits: outside the FP64 path's bounds, so AUTO
    takes the integer-pipe kernel (k_ntt_mac, two 8192-coefficient slices per
    polynomial); ciphertexts and decryption against the oracle, 2 batches + ragged."""
    base = inp.CONFIGS["c4"]
    cfg = dataclasses.replace(base, name="c4q55", q_bits=(55,) * 9, D_live=512, D_stored=512, nq=2 * 2340 + 77)
    nq = cfg.nq
    Xtr, ytr, Xq, _ = inp.gen_features(cfg)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, deterministic=True)
    assert ps.ctx.arith == "int"
    assert max(ps.ctx.q) >= 1 << 50
    H, got = _run_step(ps, cfg, Xq, nq)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    H_or = opipe.encode_queries(om, P, Xq)
    assert np.array_equal(H, H_or)
    want = opipe.infer_all(om, H_or)
    assert np.array_equal(got, want)
    S, lab = eph.decrypt_scores(ps.ctx, ps.sk, got, nq)
    Sref = hdc.scores(H_or, om.class_hv)
    assert np.array_equal(S, Sref)
    assert np.array_equal(lab.astype(np.int64), hdc.argmax_lowest(Sref))
