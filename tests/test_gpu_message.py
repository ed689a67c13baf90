"""Scores message on the GPU (NEXT #4; -m gpu): the device bit-packing equals the
oracle's plain packer byte for byte, the host unpacker inverts it, and the end-to-end
packed client call returns the message of the device path's ciphertexts."""
import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import message

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_00737_b200 as eph  # noqa: E402
from paper_2511_00737_b200 import pipeline as ppipe  # noqa: E402


@pytest.mark.parametrize("name,nq", [("c1q3", 700), ("c2", 2100), ("c3", 900)])
def test_message_bitexact(name, nq):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    ps = ppipe.build(cfg, inp.gen_projection(cfg), Xtr, ytr, deterministic=True)
    ctx = ps.ctx
    ws = eph.Workspace(ctx, nq)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    cts = eph.infer_batch(ctx, ps.model, ws, eph.encode_queries(ctx, X, ps.P_dev), nq)
    msg = eph.pack_scores(ctx, cts)
    torch.cuda.synchronize()
    ct_h = cts.cpu().numpy().view(np.uint64)
    nb = ct_h.shape[0]
    got = msg.cpu().numpy().tobytes()
    assert len(got) == eph.scores_message_bytes(ctx, nb) == message.message_bytes(nb, ctx.N, ctx.q)
    assert got == message.pack(ct_h, ctx.q)
    assert np.array_equal(eph.unpack_scores(ctx, np.frombuffer(got, np.uint8), nb), ct_h)
    Xh = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).pin_memory()
    e2e = eph.classify_host_packed(ctx, ps.model, ws, Xh, ps.P_dev)
    assert e2e.numpy().tobytes() == got
