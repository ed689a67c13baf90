"""The C-ABI library loads, exports every symbol of include/ephdc.h, and its host-only
entry points (primes, psi, CDT, keygen, decryption) agree with the oracle (not gpu).
No compute kernel is called here."""
import os
import re

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import hdc, nt, pipeline as opipe
from oracle.bfv import OracleBFV, gaussian_cdt as oracle_cdt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import paper_2511_00737_b200 as eph  # noqa: E402
from paper_2511_00737_b200 import _capi  # noqa: E402


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "ephdc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ephdc_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    syms = _header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(_capi.lib, s), s
    assert set(syms) == set(_capi.EXPORTED)
    assert _capi.lib.ephdc_abi_version() == 4


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if line.strip())


@pytest.mark.parametrize("name", ["c1", "c1q3", "c2", "c3", "c4"])
def test_primes_and_psi_match_oracle(name):
    cfg = inp.CONFIGS[name]
    t_or = nt.plaintext_modulus(cfg.t_bits, cfg.log2N, cfg.t_fixed)
    q_or = nt.prime_chain(cfg.q_bits, cfg.log2N, exclude=[t_or])
    if cfg.t_fixed is None:
        assert eph.find_ntt_primes(cfg.log2N, [cfg.t_bits]) == [t_or]
    assert eph.find_ntt_primes(cfg.log2N, cfg.q_bits, exclude=[t_or]) == q_or
    for p in [t_or] + q_or:
        assert eph.min_psi(p, cfg.log2N) == nt.min_primitive_2n_root(p, cfg.N)


def test_c5_prime_availability():
    # 16 primes of 30 and 60 bits exist at every c5 ring degree (BASELINE.json configs[4])
    for lg in inp.C5_LOG2N:
        for bits in inp.C5_WORD_BITS:
            ps = eph.find_ntt_primes(lg, [bits] * 16)
            assert len(set(ps)) == 16 and all(p % (2 << lg) == 1 for p in ps)
            assert ps == nt.prime_chain([bits] * 16, lg)


def test_bad_params_rejected():
    with pytest.raises(eph.EphdcError):
        eph.find_ntt_primes(10, [11])          # 2^11 <= 2N: no prime of that form below it
    with pytest.raises(eph.EphdcError):
        eph.min_psi(65539, 10)                 # not = 1 mod 2N


def test_gaussian_cdt_matches_oracle():
    assert np.array_equal(eph.gaussian_cdt(3.2), oracle_cdt(3.2))


def _host_ctx(name, Qbits=None, qshift=0):
    cfg = inp.CONFIGS[name]
    bfv = OracleBFV(cfg)
    Q = Qbits or hdc.choose_Qbits(cfg.D_live, cfg.Cbits, bfv.t)
    ctx = eph.Context(log2N=cfg.log2N, q=bfv.q, t=bfv.t, k=cfg.k, D_live=cfg.D_live, D_stored=cfg.D_stored,
                      F=cfg.F, feat_unsigned=cfg.feat_unsigned, Qbits=Q, Cbits=cfg.Cbits, qshift=qshift,
                      sigma_e=cfg.sigma_e, device=-1)
    return cfg, bfv, ctx


@pytest.mark.parametrize("name", ["c1q3", "c2", "c3", "c4"])
def test_host_context_derived_values(name):
    cfg, bfv, ctx = _host_ctx(name)
    assert ctx.B == bfv.B and ctx.t == bfv.t and ctx.q == bfv.q
    assert ctx.psi_t == bfv.psi_t and ctx.psi == bfv.psi
    assert ctx.delta == bfv.delta
    assert ctx.info.device == -1


def test_context_validation():
    cfg, bfv, _ = _host_ctx("c1q3")
    base = dict(log2N=10, q=bfv.q, t=bfv.t, k=2, D_live=1024, D_stored=1024, F=64, feat_unsigned=False,
                Qbits=3, Cbits=4, qshift=0, device=-1)
    for bad in (dict(t=65539), dict(q=[bfv.q[0], bfv.q[0]]), dict(F=62), dict(log2N=9), dict(Qbits=9),
                dict(D_stored=10), dict(q=[65537 * 0 + 12289])):
        kw = dict(base)
        kw.update(bad)
        with pytest.raises(eph.EphdcError):
            eph.Context(**kw)


@pytest.mark.parametrize("name", ["c1q3", "c2", "c4"])
def test_keygen_matches_oracle(name):
    cfg, bfv, ctx = _host_ctx(name)
    sk = eph.SecretKey(ctx, 1234)
    s, sh = sk.export()
    assert np.array_equal(s, bfv.keygen(1234))
    assert np.array_equal(sh, bfv.s_hat)


def test_chacha20_block_known_answers():
    """The library's generator (rng.cuh, host side) against RFC 8439's known answers."""
    import json, os, struct
    gold = os.path.join(os.path.dirname(__file__), "golden", "chacha20_kat.json")
    for v in json.load(open(gold))["vectors"]:
        nonce = struct.unpack("<3I", bytes.fromhex(v["nonce"]))
        want = np.array(struct.unpack("<16I", bytes.fromhex(v["block"])), dtype=np.uint32)
        assert np.array_equal(eph.chacha20_block(bytes.fromhex(v["key"]), v["counter"], nonce), want), v["source"]


def test_keys_default_to_os_entropy():
    """No seed: every key is fresh (ephdc_seed_os); an int seed is the deterministic test key."""
    _, bfv, ctx = _host_ctx("c1q3")
    s1, s2 = eph.SecretKey(ctx).export()[0], eph.SecretKey(ctx).export()[0]
    assert not np.array_equal(s1, s2)
    for s in (s1, s2):
        assert set(np.unique(s)) <= {-1, 0, 1} and abs((s == 0).mean() - 1 / 3) < 0.1
    key = (1234).to_bytes(8, "little") + bytes(24)     # ephdc_seed_u64(v) = (lo32, hi32, 0, ..., 0)
    assert np.array_equal(eph.SecretKey(ctx, key).export()[0], bfv.keygen(1234))
    with pytest.raises(ValueError):
        eph.make_seed(b"short")


@pytest.mark.parametrize("name,nq", [("c1q3", 700), ("c2", 300)])
def test_decrypt_scores_matches_oracle(name, nq):
    cfg = inp.CONFIGS[name]
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, nq)
    P = inp.gen_projection(cfg)
    om = opipe.build_model(cfg, P, Xtr, ytr)
    H = opipe.encode_queries(om, P, Xq)
    cts = opipe.infer_all(om, H)
    _, _, ctx = _host_ctx(name, om.Qbits, om.qshift)
    sk = eph.SecretKey(ctx, om.sk_seed)
    S, lab = eph.decrypt_scores(ctx, sk, cts, nq)
    Sref = hdc.scores(H, om.class_hv)
    assert np.array_equal(S, Sref)
    assert np.array_equal(lab.astype(np.int64), hdc.argmax_lowest(Sref))
    slots = eph.decrypt_slots(ctx, sk, cts[0])
    assert np.array_equal(slots, om.bfv.decrypt(cts[0]))


def test_product_model_build_matches_oracle():
    for name in ("c1q3", "c2", "c3"):
        cfg = inp.CONFIGS[name]
        Xtr, ytr, _, _ = inp.gen_features(cfg, 8)
        P = inp.gen_projection(cfg)
        bfv = OracleBFV(cfg)
        Q = hdc.choose_Qbits(cfg.D_live, cfg.Cbits, bfv.t)
        assert eph.query_bits(cfg.D_live, cfg.Cbits, bfv.t) == Q
        acc = hdc.encode_raw(P, Xtr, cfg.D_live)   # input to both sides
        C, s = eph.train_model(acc, ytr, cfg.k, cfg.Cbits, Q)
        assert s == hdc.calibrate_shift(acc, Q)
        assert np.array_equal(C, hdc.quantise_classes(hdc.bundle(acc, ytr, cfg.k), cfg.Cbits))
