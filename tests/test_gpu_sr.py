"""HE-HDC-SR on the GPU (NEXT #3; -m gpu): the client's query ciphertexts and the
server's evaluation equal the oracle's bit-exactly and decrypt to the brute-force dot
products, on both arithmetic paths."""
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


@pytest.mark.parametrize("name,nq,arith", [("c1q3", 700, 0), ("c2", 300, 0), ("c2", 300, 1)])
def test_sr_bitexact(name, nq, arith):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, arith=arith, deterministic=True)
    ctx = ps.ctx
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    H = eph.encode_queries(ctx, X, ps.P_dev)
    ws = eph.Workspace(ctx, nq)
    pt = eph.sr_model_plaintexts(ctx, ps.class_hv)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    H_or = opipe.encode_queries(om, P, Xq)
    Sref = hdc.scores(H_or, om.class_hv)
    for b in range(ctx.n_batches(nq)):
        qct = eph.sr_encrypt_queries(ctx, ps.sk, ws, H, nq, b, seed=4242)
        res = eph.sr_evaluate(ctx, pt, qct)
        torch.cuda.synchronize()
        want_q = om.bfv.sr_encrypt_queries(H_or, nq, b, enc_seed=4242)
        assert np.array_equal(qct.cpu().numpy().view(np.uint64), want_q)
        got = res.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, om.bfv.sr_server_eval(om.class_hv, want_q))
        nb = min(ctx.B, nq - b * ctx.B)
        v = eph.decrypt_slots(ctx, ps.sk, got).astype(np.int64)
        v = np.where(v > (ctx.t - 1) // 2, v - ctx.t, v)
        assert np.array_equal(v[: ctx.k * nb].reshape(nb, ctx.k), Sref[b * ctx.B: b * ctx.B + nb])
