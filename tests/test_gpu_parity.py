"""GPU parity of the C-ABI hot path against the CPU oracle (bit-exact; -m gpu).

Both sides read the same seeded inputs (ephdc_inputs); the product trains, keys and
encrypts with its own code (library kernels + host C++), the oracle with its own.
Compared bit-exactly: class HVs and query shift, encoded hypervectors H, model
ciphertexts, plaintext NTTs, scores ciphertexts; decrypted scores must equal the
brute-force integer dot products and labels their argmax (north_star).
"""
import os

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

_CACHE = {}


ARITH = {"auto": 0, "int": 1, "f64": 2}


def setup(name, nq, arith="auto"):
    key = (name, nq, arith)
    if key in _CACHE:
        return _CACHE[key]
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, yq = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    ps = ppipe.build(cfg, P, Xtr, ytr, arith=ARITH[arith], deterministic=True)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    H_dev = eph.encode_queries(ps.ctx, X, ps.P_dev)
    torch.cuda.synchronize()
    H_or = opipe.encode_queries(om, P, Xq)
    r = dict(cfg=cfg, om=om, ps=ps, P=P, Xq=Xq, yq=yq, X=X, H_dev=H_dev, H_or=H_or, nq=nq)
    _CACHE[key] = r
    return r


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


CASES = [("c1", 16, "auto"), ("c1q3", 16, "auto"), ("c1q3", 700, "auto"), ("c2", 1024, "auto"), ("c2", 2100, "auto"),
         ("c3", 900, "auto"),
         # the integer-pipe kernel (used when a prime is >= 2^50) on the same workloads
         ("c1q3", 700, "int"), ("c2", 2100, "int"), ("c3", 900, "int")]


def test_arith_selection():
    # every BASELINE.json config has primes < 2^50: AUTO selects the FP64 pipe;
    # c4 (48-bit primes, N = 16384) needs the mid-NTT reduction
    for name in ("c1", "c1q3", "c2", "c3"):
        r = setup(name, 16)
        assert r["ps"].ctx.arith == "f64", name
        assert r["ps"].ctx.info.f64_red_every >= 1
    assert setup("c2", 2100, "int")["ps"].ctx.arith == "int"


@pytest.mark.parametrize("name,nq,arith", CASES)
def test_model_build_and_encoding_bitexact(name, nq, arith):
    r = setup(name, nq, arith)
    assert r["ps"].Qbits == r["om"].Qbits and r["ps"].qshift == r["om"].qshift
    assert np.array_equal(r["ps"].class_hv, r["om"].class_hv)
    assert np.array_equal(r["H_dev"].cpu().numpy(), r["H_or"])


@pytest.mark.parametrize("name,nq", [("c1", 16), ("c1q3", 16), ("c2", 1024), ("c3", 900)])
def test_model_ciphertexts_bitexact(name, nq):
    r = setup(name, nq)
    D = r["cfg"].D_live
    for d0, nd in ((0, 3), (D // 2, 2), (D - 3, 3)):
        got = r["ps"].model.export(d0, nd)
        want = r["om"].bfv.encrypt_dims(r["om"].class_hv, r["om"].enc_seed, d0, nd)
        assert np.array_equal(got, want), (d0, nd)


@pytest.mark.parametrize("name,nq,arith", [("c1q3", 700, "auto"), ("c2", 2100, "auto"), ("c3", 900, "auto"),
                                          ("c2", 2100, "int"), ("c3", 900, "int")])
def test_plaintext_ntts_bitexact(name, nq, arith):
    r = setup(name, nq, arith)
    ps, om = r["ps"], r["om"]
    ws = eph.Workspace(ps.ctx, nq)
    nb = ps.ctx.n_batches(nq)
    for b in sorted({0, nb - 1}):
        for d0 in (0, r["cfg"].D_live - 4):
            got = _u64(eph.encode_plaintexts(ps.ctx, ws, r["H_dev"], b, d0, 4))
            want = om.bfv.plaintext_ntts(r["H_or"], nq, b, d0, 4)
            assert np.array_equal(got, want), (b, d0)


@pytest.mark.parametrize("name,nq,arith", CASES)
def test_infer_bitexact_and_decrypts_to_dot_products(name, nq, arith):
    r = setup(name, nq, arith)
    ps, om = r["ps"], r["om"]
    ws = eph.Workspace(ps.ctx, nq)
    cts = eph.infer_batch(ps.ctx, ps.model, ws, r["H_dev"], nq)
    torch.cuda.synchronize()
    got = _u64(cts)
    cfg = r["cfg"]
    model = om.bfv.encrypt_dims(om.class_hv, om.enc_seed, 0, cfg.D_live) if cfg.D_live <= 4096 else None
    want = opipe.infer_all(om, r["H_or"], model=model)
    assert got.shape == want.shape
    for b in range(got.shape[0]):
        assert np.array_equal(got[b], want[b]), f"batch {b}"
    if name != "c1":          # c1 literal cannot decrypt (tests/test_oracle_bfv.py)
        S, lab = eph.decrypt_scores(ps.ctx, ps.sk, got, nq)
        Sref = hdc.scores(r["H_or"], om.class_hv)
        assert np.array_equal(S, Sref)
        assert np.array_equal(lab.astype(np.int64), hdc.argmax_lowest(Sref))


def test_edge_batches_and_errors():
    r = setup("c1q3", 16)
    ps = r["ps"]
    B = ps.ctx.B
    cfg = r["cfg"]
    _, _, Xq, _ = inp.gen_features(cfg, B + 1)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    H = eph.encode_queries(ps.ctx, X, ps.P_dev)
    ws = eph.Workspace(ps.ctx, B + 1)
    om = r["om"]
    H_or = opipe.encode_queries(om, r["P"], Xq)
    for nq in (1, B - 1, B, B + 1):
        Hn = H[:, :nq].contiguous()
        got = _u64(eph.infer_batch(ps.ctx, ps.model, ws, Hn, nq))
        S, _ = eph.decrypt_scores(ps.ctx, ps.sk, got, nq)
        assert np.array_equal(S, hdc.scores(H_or[:, :nq], om.class_hv)), nq
    out = torch.empty((1, 2, ps.ctx.L, ps.ctx.N), dtype=torch.int64, device="cuda")
    with pytest.raises(eph.EphdcError) as e:
        eph.infer_batch(ps.ctx, ps.model, ws, H, B + 1, out=out)
    assert e.value.status == 3     # EPHDC_EOVERFLOW


def test_classify_host_matches_device_path():
    r = setup("c2", 2100)
    ps = r["ps"]
    ws = eph.Workspace(ps.ctx, r["nq"])
    Xh = torch.from_numpy(np.ascontiguousarray(r["Xq"]).view(np.int8)).pin_memory()
    out_h = eph.classify_host(ps.ctx, ps.model, ws, Xh, ps.P_dev)
    dev = eph.infer_batch(ps.ctx, ps.model, ws, r["H_dev"], r["nq"])
    torch.cuda.synchronize()
    assert np.array_equal(out_h.numpy().view(np.uint64), _u64(dev))


def test_launch_counter_increases():
    r = setup("c1q3", 16)
    n0 = eph.launch_count()
    ws = eph.Workspace(r["ps"].ctx, 16)
    eph.infer_batch(r["ps"].ctx, r["ps"].model, ws, r["H_dev"], 16)
    torch.cuda.synchronize()
    assert eph.launch_count() - n0 == 3      # pack_intt, ntt_mac, finalize for one batch


@pytest.mark.parametrize("k,nq", [(1, 700), (1, 1024 + 3), (3, 341 * 2 + 5)])
def test_slot_packing_small_k(k, nq):
    """k = 1 (one query per slot: the slot -> query division is the identity) and k = 3
    (B = 341, a ragged 1024 = 3 * 341 + 1 tail slot): scores ciphertexts bit-exact with
    the oracle, decryption = brute-force dot products (k = 1)."""
    import dataclasses
    cfg = dataclasses.replace(inp.CONFIGS["c1q3"], name=f"c1q3k{k}", k=k)
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    ps = ppipe.build(cfg, P, Xtr, ytr, deterministic=True)
    X = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).cuda()
    H = eph.encode_queries(ps.ctx, X, ps.P_dev)
    ws = eph.Workspace(ps.ctx, nq)
    got = _u64(eph.infer_batch(ps.ctx, ps.model, ws, H, nq))
    H_or = opipe.encode_queries(om, P, Xq)
    assert np.array_equal(H.cpu().numpy(), H_or)
    assert np.array_equal(got, opipe.infer_all(om, H_or))
    S, lab = eph.decrypt_scores(ps.ctx, ps.sk, got, nq)
    Sref = hdc.scores(H_or, om.class_hv)
    assert np.array_equal(S, Sref)
    assert np.array_equal(lab.astype(np.int64), hdc.argmax_lowest(Sref))
