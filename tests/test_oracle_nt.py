"""Pins of the oracle's number theory (not gpu): primes, psi, bit reversal, RNG, CDT."""
import json
import math
import os
import random

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import core, nt
from oracle.bfv import gaussian_cdt

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _trial_prime(n):
    if n < 2:
        return False
    d = 2
    while d * d <= n:
        if n % d == 0:
            return False
        d += 1
    return True


def test_is_prime_matches_trial_division():
    for n in range(0, 20000):
        assert nt.is_prime(n) == _trial_prime(n), n
    # Carmichael numbers and strong pseudoprimes to small bases
    for n in (561, 1105, 1729, 2465, 2821, 6601, 8911, 3215031751, 2152302898747):
        assert not nt.is_prime(n)
    assert nt.is_prime((1 << 61) - 1)        # Mersenne prime M61
    assert not nt.is_prime((1 << 59) - 1)    # 179951 * 3203431780337


@pytest.mark.parametrize("name", ["c1", "c1q3", "c2", "c3", "c4"])
def test_prime_chain_definition(name):
    cfg = inp.CONFIGS[name]
    two_n = 2 * cfg.N
    t = nt.plaintext_modulus(cfg.t_bits, cfg.log2N, cfg.t_fixed)
    qs = nt.prime_chain(cfg.q_bits, cfg.log2N, exclude=[t])
    assert nt.is_prime(t) and t % two_n == 1
    if cfg.t_fixed is None:
        assert t < (1 << cfg.t_bits)
        # no larger candidate below the bound is prime (definition of "largest")
        c = t + two_n
        while c < (1 << cfg.t_bits):
            assert not nt.is_prime(c)
            c += two_n
    assert len(set(qs)) == len(qs) and t not in qs
    used = [t]
    for b, q in zip(cfg.q_bits, qs):
        assert nt.is_prime(q) and q % two_n == 1 and q < (1 << b)
        c = q + two_n
        while c < (1 << b):
            assert (not nt.is_prime(c)) or c in used, (b, c)
            c += two_n
        used.append(q)


def test_min_psi_bruteforce_small():
    for logN in (2, 3, 4, 5):
        N = 1 << logN
        for p in [x for x in range(3, 4000) if _trial_prime(x) and x % (2 * N) == 1]:
            brute = next(x for x in range(2, p) if pow(x, N, p) == p - 1)
            assert nt.min_primitive_2n_root(p, N) == brute


@pytest.mark.parametrize("name", ["c1q3", "c2", "c3", "c4"])
def test_psi_is_primitive_and_minimal(name):
    cfg = inp.CONFIGS[name]
    N = cfg.N
    t = nt.plaintext_modulus(cfg.t_bits, cfg.log2N, cfg.t_fixed)
    for p in [t] + nt.prime_chain(cfg.q_bits, cfg.log2N, exclude=[t]):
        psi = nt.min_primitive_2n_root(p, N)
        assert pow(psi, N, p) == p - 1            # order exactly 2N (2N a power of two)
        # every primitive 2N-th root is an odd power of psi; none is smaller
        sq = psi * psi % p
        x = psi
        for _ in range(N - 1):
            x = x * sq % p
            assert x >= psi


def test_brev():
    assert [nt.brev(i, 3) for i in range(8)] == [0, 4, 2, 6, 1, 5, 3, 7]
    L = core.lib()
    for bits in (1, 5, 10, 14):
        for i in random.Random(1).sample(range(1 << bits), min(200, 1 << bits)):
            assert L.or_brev(i, bits) == nt.brev(i, bits)
            assert nt.brev(nt.brev(i, bits), bits) == i


def _kat_vectors():
    import struct
    for v in json.load(open(os.path.join(GOLD, "chacha20_kat.json")))["vectors"]:
        key = np.array(struct.unpack("<8I", bytes.fromhex(v["key"])), dtype=np.uint32)
        nonce = np.array(struct.unpack("<3I", bytes.fromhex(v["nonce"])), dtype=np.uint32)
        want = np.array(struct.unpack("<16I", bytes.fromhex(v["block"])), dtype=np.uint32)
        yield v, key, nonce, want


def test_chacha20_known_answers():
    """RFC 8439 sec. 2.3.2 and A.1 #1 pin the oracle's block function (reading #7)."""
    L = core.lib()
    for v, key, nonce, want in _kat_vectors():
        out = np.zeros(16, dtype=np.uint32)
        L.or_chacha20_block(core.ptr(key), v["counter"], core.ptr(nonce), core.ptr(out))
        assert np.array_equal(out, want), v["source"]


def test_word64_is_block_word():
    """or_word64 = little-endian word w of the block under key (lo, hi, 0..0), nonce (tag, a)."""
    L = core.lib()
    seed, tag, a = 0x0123456789ABCDEF, 3, (7 << 32) | 11
    key = np.array([seed & 0xFFFFFFFF, seed >> 32, 0, 0, 0, 0, 0, 0], dtype=np.uint32)
    nonce = np.array([tag, a & 0xFFFFFFFF, a >> 32], dtype=np.uint32)
    for ctr in (0, 5):
        b = np.zeros(16, dtype=np.uint32)
        L.or_chacha20_block(core.ptr(key), ctr, core.ptr(nonce), core.ptr(b))
        for w in range(8):
            assert L.or_word64(seed, tag, a, ctr, w) == int(b[2 * w]) | (int(b[2 * w + 1]) << 32)


def test_uniform_rejection_path():
    """q just above a power of two: about half the first draws are rejected, the retry
    stream fills them, and the result is still uniform on [0, q)."""
    L = core.lib()
    q = (1 << 20) + 7                     # mask = 2^21 - 1
    N = 1 << 14
    a = np.array([L.or_uniform_mod(9, 4, 1, 3, i, q) for i in range(N)], dtype=np.int64)
    assert a.max() < q and a.min() >= 0
    first = np.array([L.or_word64(9, 3, 4 * 3 + 1, i // 8, i % 8) & ((1 << 21) - 1) for i in range(N)])
    acc = first < q
    assert 0.4 < acc.mean() < 0.6
    assert np.array_equal(a[acc], first[acc])          # accepted first draws are kept as drawn
    assert abs(a.mean() / q - 0.5) < 0.02 and abs(a[~acc].mean() / q - 0.5) < 0.03


def test_gaussian_cdt_pins():
    T = gaussian_cdt(3.2)
    assert T.dtype == np.uint64 and len(T) == 20
    assert int(T[-1]) == 1 << 63
    assert all(int(T[i]) < int(T[i + 1]) for i in range(19))
    # closed form in float: p(0) = 1/Z, cdf(k) = (1 + 2 sum_{1..k} rho)/Z
    rho = [math.exp(-k * k / (2 * 3.2 ** 2)) for k in range(20)]
    Z = rho[0] + 2 * sum(rho[1:])
    for k in range(19):
        cdf = (rho[0] + 2 * sum(rho[1:k + 1])) / Z
        assert abs(int(T[k]) / 2.0 ** 63 - cdf) < 2 ** -39
    # rounding margin: no entry sits near a rounding boundary of the 2^40 grid,
    # so any correct independent evaluation rounds identically
    from decimal import Decimal, getcontext
    getcontext().prec = 50
    s = Decimal("3.2")
    rd = [(-(Decimal(k) ** 2) / (2 * s * s)).exp() for k in range(20)]
    Zd = rd[0] + 2 * sum(rd[1:])
    for k in range(19):
        v = (rd[0] + 2 * sum(rd[1:k + 1])) / Zd * (Decimal(2) ** 40)
        frac = v - int(v)
        assert abs(frac - Decimal("0.5")) > Decimal("0.01")


def test_sampler_statistics():
    L = core.lib()
    N = 1 << 14
    s = np.empty(N, dtype=np.int8)
    L.or_sample_ternary(99, N, core.ptr(s))
    assert set(np.unique(s)) <= {-1, 0, 1}
    for v in (-1, 0, 1):
        assert abs((s == v).mean() - 1 / 3) < 0.02
    T = np.ascontiguousarray(gaussian_cdt(3.2))
    e = np.empty(N, dtype=np.int64)
    L.or_sample_gauss_poly(7, 3, N, core.ptr(T), 20, core.ptr(e))
    assert abs(e.mean()) < 0.1 and abs(e.std() - 3.2) < 0.1 and np.abs(e).max() <= 19
    q = 281474976546817
    a = np.empty(N, dtype=np.uint64)
    L.or_sample_uniform_poly(5, 2, 1, 9, q, N, core.ptr(a))
    assert int(a.max()) < q
    assert abs(a.astype(np.float64).mean() / q - 0.5) < 0.02


def test_poly_samplers_match_coefficient_samplers():
    """or_sample_*_poly (one block per 8 / 4 coefficients) = the per-coefficient definitions."""
    L = core.lib()
    N = 1 << 10
    for q in ((1 << 20) + 7, 281474976546817):
        a = np.empty(N, dtype=np.uint64)
        L.or_sample_uniform_poly(11, 6, 2, 5, q, N, core.ptr(a))
        assert [int(v) for v in a] == [L.or_uniform_mod(11, 6, 2, 5, i, q) for i in range(N)]
    T = np.ascontiguousarray(gaussian_cdt(3.2))
    e = np.empty(N, dtype=np.int64)
    L.or_sample_gauss_poly(11, (1 << 32) + 3, N, core.ptr(T), 20, core.ptr(e))
    assert [int(v) for v in e] == [L.or_gauss(11, (1 << 32) + 3, i, core.ptr(T), 20) for i in range(N)]
