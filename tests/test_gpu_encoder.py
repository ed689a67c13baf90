"""HDC encoding GEMM on the GPU vs the oracle, bit-exact (-m gpu):
the tcgen05 kind::i8 tensor-core kernel (default) and the dp4a CUDA-core kernel
(ephdc_params.encoder = 1), quantised and raw epilogues, ragged query counts
(tiles of 128), F below one 128-byte K tile (c1: F = 64) and uint8 features (c3)."""
import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import hdc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2511_00737_b200 as eph  # noqa: E402
from paper_2511_00737_b200 import pipeline as ppipe  # noqa: E402


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
@pytest.mark.parametrize("encoder", [0, 1])
@pytest.mark.parametrize("nq", [1, 127, 129, 300])
def test_encoder_bitexact(name, encoder, nq):
    cfg = inp.CONFIGS[name]
    _, _, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    t, q = ppipe.primes_for(cfg)
    Qbits, shift = 5, 7
    ctx = ppipe.make_context(cfg, t, q, Qbits, shift, device=0, encoder=encoder)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    Pd = torch.from_numpy(np.ascontiguousarray(P)).cuda()
    acc_ref = hdc.encode_raw(P, Xq, cfg.D_live)
    raw = eph.encode_raw(ctx, X, Pd).cpu().numpy()
    assert np.array_equal(raw, acc_ref)
    H = eph.encode_queries(ctx, X, Pd).cpu().numpy()
    assert np.array_equal(H, hdc.quantise_queries(acc_ref, shift, Qbits))
