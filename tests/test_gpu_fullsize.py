"""Full-size parity in the launch configuration bench.py times (-m gpu).

BASELINE.json configs[2] (c3, 8192 queries = 11 batches) and configs[3] (c4, 65536
queries = 29 batches, N = 16384, 9 x 48-bit primes): the whole step runs through the
same calls bench.py times (encode_queries + infer_batch over every batch, one fused
launch).  Checked against the oracle:
  * H (all queries) bit-exact;
  * scores ciphertexts of sampled batches (first, middle, last = ragged) bit-exact
    against the oracle's own evaluation (its own model encryption on the fly);
  * EVERY batch decrypts to the brute-force integer dot products, every label is the
    lowest-index argmax (a property that holds at any size).
"""
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


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_fullsize_step_parity(name):
    cfg = inp.CONFIGS[name]
    nq = cfg.nq
    Xtr, ytr, Xq, _ = inp.gen_features(cfg)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr)
    assert ps.ctx.arith == "f64"
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    ws = eph.Workspace(ps.ctx, nq)
    H = torch.empty((cfg.D_live, nq), dtype=torch.int8, device="cuda")
    out = torch.empty(ps.ctx.ct_shape(nq), dtype=torch.int64, device="cuda")
    eph.encode_queries(ps.ctx, X, ps.P_dev, H)
    eph.infer_batch(ps.ctx, ps.model, ws, H, nq, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint64)
    nb = got.shape[0]

    om = opipe.build_model(cfg, P, Xtr, ytr)
    assert np.array_equal(ps.class_hv, om.class_hv)
    H_or = opipe.encode_queries(om, P, Xq)
    assert np.array_equal(H.cpu().numpy(), H_or)
    for b in sorted({0, nb // 2, nb - 1}):
        want = om.bfv.infer_batch(H_or, nq, b, class_hv=om.class_hv, enc_seed=om.enc_seed)
        assert np.array_equal(got[b], want), f"batch {b}"

    S, lab = eph.decrypt_scores(ps.ctx, ps.sk, got, nq)
    Sref = hdc.scores(H_or, om.class_hv)
    assert np.array_equal(S, Sref)
    assert np.array_equal(lab.astype(np.int64), hdc.argmax_lowest(Sref))
