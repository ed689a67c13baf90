"""Accumulator scaling on the GPU (NEXT #1) vs the oracle's literal
sequential procedure, bit-exact (-m gpu).  ephdc_model_scale folds the schedule into
the encrypted model; infer_batch must then return the ciphertexts of
acc <- (acc + sum_{d in J} CT_d PT_d) * s_J^-1, on both arithmetic paths."""
import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import pipeline as opipe

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_00737_b200 as eph  # noqa: E402
from paper_2511_00737_b200 import pipeline as ppipe  # noqa: E402


@pytest.mark.parametrize("name,nq,g,scales,arith", [
    ("c1q3", 700, 512, [256, 256], 0),
    ("c1q3", 700, 300, [4096, 16384, 256, 4096], 0),
    ("c1q3", 700, 300, [4096, 16384, 256, 4096], 1),
    ("c2", 300, 512, [1] * 8, 0),
    ("c2", 300, 1000, [2, 1, 1, 4, 1], 0),
])
def test_scaled_model_matches_sequential_oracle(name, nq, g, scales, arith):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, arith=arith, deterministic=True)
    ps.model.scale(g, scales)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    H = eph.encode_queries(ps.ctx, X, ps.P_dev)
    ws = eph.Workspace(ps.ctx, nq)
    got = eph.infer_batch(ps.ctx, ps.model, ws, H, nq).cpu().numpy().view(np.uint64)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    H_or = opipe.encode_queries(om, P, Xq)
    for b in range(got.shape[0]):
        want = om.bfv.infer_batch_scaled(H_or, nq, b, g, scales, class_hv=om.class_hv, enc_seed=om.enc_seed)
        assert np.array_equal(got[b], want), b


def test_model_scale_rejects_bad_schedules():
    cfg = inp.CONFIGS["c1q3"]
    Xtr, ytr, _, _ = inp.gen_features(cfg, 4)
    ps = ppipe.build(cfg, inp.gen_projection(cfg), Xtr, ytr, deterministic=True)
    for g, scales in ((512, [1]), (0, []), (512, [1, 65537])):
        with pytest.raises(eph.EphdcError) as e:
            ps.model.scale(g, scales)
        assert e.value.status == 1      # EPHDC_EPARAM
