"""Launch-plan variants of the fused FP64 kernel give bit-identical ciphertexts (-m gpu).

The default plan (f64_grid + the WL / prefetch choice in mac_f64_launch) is checked
against the oracle by test_gpu_fullsize / test_gpu_parity; every other variant the
workspace plan overrides (ephdc_plan) select must produce exactly the same scores ciphertexts:
the two-group kernel (the NC = 2^13 default) against the one-team kernel, the round-1
slot pack + INTT_t kernel against the ntt32_c5.cu one, the
synchronisation variants WL = 0/1/2, 32 elements per thread, the explicit L2
prefetch on/off, and other grid plans (batches per group, dims per chunk -- i.e. other
orders of the 64-bit atomic folds, which integer addition makes order independent).
Each variant's output also decrypts to the brute-force integer scores.
"""
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

VARIANTS = [
    {"flags": 2},            # WL = 0: a CTA barrier after every pass
    {"flags": 6},            # WL = 1
    {"flags": 4},            # WL = 2
    {"flags": 16},           # explicit L2 prefetch on
    {"flags": 1},            # explicit L2 prefetch off
    {"flags": 8},            # 32 elements per thread (NC = 2^13 only), planned WL
    {"flags": 14},           # 32 elements per thread, WL = 1
    {"flags": 12},           # 32 elements per thread, WL = 2
    {"flags": 32},           # the one-team kernel (default plan) at NC = 2^13
    {"bg": 1, "G": 37},      # (two groups) odd chunks: the groups' dims and tokens
    {"bg": 2, "G": 1000},
    {"bg": 3, "G": 9},       # chunks of 9 dims (the planner's minimum at c3 is 8)
    {"flags": 32, "G": 37},
    {"flags": 64},           # the two-group kernel at N = 2^14 (c4; one team by default)
    {"flags": 64, "bg": 1, "G": 37},
    {"flags": 128},          # the round-1 slot pack + INTT_t kernel (default: ntt32_c5.cu passes)
    {"flags": 256},          # the ntt32_c5.cu pack without the next-row prefetch
]


def _run(ps, H, nq, plan):
    ws = eph.Workspace(ps.ctx, nq, plan=plan)
    out = eph.infer_batch(ps.ctx, ps.model, ws, H, nq)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint64).copy()


@pytest.mark.parametrize("name,extra", [("c3", 77), ("c4", 123)])
def test_plan_variants_bit_identical(name, extra):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, deterministic=True)
    assert ps.ctx.arith == "f64"
    nq = 2 * ps.ctx.B + extra                      # 3 batches, the last ragged
    Xs = np.ascontiguousarray(Xq[:nq])
    X = torch.from_numpy(Xs.view(np.int8)).cuda()
    H = eph.encode_queries(ps.ctx, X, ps.P_dev)
    ref = _run(ps, H, nq, None)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    H_or = opipe.encode_queries(om, P, Xs)
    Sref = hdc.scores(H_or, om.class_hv)
    S, _ = eph.decrypt_scores(ps.ctx, ps.sk, ref, nq)
    assert np.array_equal(S, Sref)
    for plan in VARIANTS:
        got = _run(ps, H, nq, plan)
        assert np.array_equal(got, ref), plan


@pytest.mark.parametrize("name,groups", [("c3", 2), ("c4", 7)])
def test_batch_groups_bit_identical(name, groups):
    """The FP64 path packs and evaluates the batches of a call in groups of at most
    m_batches (the plaintext workspace is capped at 32 GB; c4 beyond ~50 batches):
    grouping changes only the launch boundaries, never the ciphertexts."""
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, deterministic=True)
    nq = 5 * ps.ctx.B + 11 if name == "c3" else 15 * ps.ctx.B + 7
    X = torch.from_numpy(np.ascontiguousarray(Xq[:nq]).view(np.int8)).cuda()
    H = eph.encode_queries(ps.ctx, X, ps.P_dev)
    ref = eph.infer_batch(ps.ctx, ps.model, eph.Workspace(ps.ctx, nq), H, nq).cpu().numpy()
    ws = eph.Workspace(ps.ctx, nq, plan={"m_batches": groups})
    got = eph.infer_batch(ps.ctx, ps.model, ws, H, nq).cpu().numpy()
    assert np.array_equal(got, ref)
