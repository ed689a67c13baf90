"""Pins of the oracle's negacyclic NTT and slot codec (not gpu).

The NTT output index i must equal the evaluation a(psi^(2*brev(i)+1)) (reading #1);
pinned by pure-Python direct evaluation (O(N^2)) at tiny N, by Horner evaluation at
sampled points at full N, by the convolution theorem against a pure-Python schoolbook
product in Z_q[X]/(X^N+1), and by the SPEC examples.
"""
import random

import numpy as np
import pytest

import ephdc_inputs as inp
from oracle import core, nt
from oracle.bfv import OracleBFV

SMALL_PRIMES = [(3, 97), (4, 97), (5, 193), (6, 257), (6, 7681)]


def direct_eval(a, q, x):
    return sum(int(c) * pow(x, n, q) for n, c in enumerate(a)) % q


def schoolbook(a, b, q):
    N = len(a)
    c = [0] * N
    for i in range(N):
        for j in range(N):
            p = int(a[i]) * int(b[j])
            if i + j < N:
                c[i + j] += p
            else:
                c[i + j - N] -= p
    return np.array([v % q for v in c], dtype=np.uint64)


@pytest.mark.parametrize("logN,q", SMALL_PRIMES)
def test_ntt_equals_direct_evaluation_small(logN, q):
    N = 1 << logN
    psi = nt.min_primitive_2n_root(q, N)
    rng = np.random.default_rng(logN)
    for _ in range(3):
        a = rng.integers(0, q, size=N, dtype=np.uint64)
        A = core.ntt_fwd(a, logN, q, psi)
        for i in range(N):
            assert int(A[i]) == direct_eval(a, q, pow(psi, 2 * nt.brev(i, logN) + 1, q))
        assert np.array_equal(core.ntt_inv(A, logN, q, psi), a)


@pytest.mark.parametrize("logN,q", SMALL_PRIMES)
def test_convolution_theorem_small(logN, q):
    N = 1 << logN
    psi = nt.min_primitive_2n_root(q, N)
    rng = np.random.default_rng(100 + logN)
    a = rng.integers(0, q, size=N, dtype=np.uint64)
    b = rng.integers(0, q, size=N, dtype=np.uint64)
    A = core.ntt_fwd(a, logN, q, psi)
    Bh = core.ntt_fwd(b, logN, q, psi)
    prod = np.array([int(x) * int(y) % q for x, y in zip(A, Bh)], dtype=np.uint64)
    assert np.array_equal(core.ntt_inv(prod, logN, q, psi), schoolbook(a, b, q))
    assert np.array_equal(core.negacyclic_mul(a, b, q), schoolbook(a, b, q))


@pytest.mark.parametrize("name", ["c1q3", "c2", "c3", "c4"])
def test_ntt_full_size_horner_and_spec_examples(name):
    bfv = OracleBFV(inp.CONFIGS[name])
    logN, N = bfv.logN, bfv.N
    rng = np.random.default_rng(7)
    pts = random.Random(3).sample(range(N), 16)
    for q, psi in list(zip(bfv.q, bfv.psi))[:2] + [(bfv.t, bfv.psi_t)]:
        a = rng.integers(0, q, size=N, dtype=np.uint64)
        A = core.ntt_fwd(a, logN, q, psi)
        coeffs = [int(c) for c in a]
        for i in pts:
            x = pow(psi, 2 * nt.brev(i, logN) + 1, q)
            r = 0
            for c in reversed(coeffs):       # pure-Python Horner
                r = (r * x + c) % q
            assert int(A[i]) == r
        assert np.array_equal(core.ntt_inv(A, logN, q, psi), a)          # S:48 roundtrip
        delta = np.zeros(N, dtype=np.uint64)
        delta[0] = 1
        assert np.all(core.ntt_fwd(delta, logN, q, psi) == 1)
        x1 = np.zeros(N, dtype=np.uint64); x1[1] = 1
        xn = np.zeros(N, dtype=np.uint64); xn[N - 1] = 1
        p = (core.ntt_fwd(x1, logN, q, psi).astype(object) * core.ntt_fwd(xn, logN, q, psi).astype(object)) % q
        r = core.ntt_inv(np.array(p, dtype=np.uint64), logN, q, psi)
        assert int(r[0]) == q - 1 and np.all(r[1:] == 0)                 # X * X^(N-1) = -1


def test_x_plus_1_times_x_minus_1():
    # (X+1)(X-1) = X^2 - 1
    q, logN = 7681, 4
    N = 1 << logN
    a = np.zeros(N, np.uint64); a[0] = 1; a[1] = 1
    b = np.zeros(N, np.uint64); b[0] = q - 1; b[1] = 1
    c = core.negacyclic_mul(a, b, q)
    want = np.zeros(N, np.uint64); want[0] = q - 1; want[2] = 1
    assert np.array_equal(c, want)


@pytest.mark.parametrize("name", ["c1q3", "c2"])
def test_slot_codec(name):
    bfv = OracleBFV(inp.CONFIGS[name])
    t, N = bfv.t, bfv.N
    rng = np.random.default_rng(11)
    v = rng.integers(0, t, size=N, dtype=np.uint64)
    w = rng.integers(0, t, size=N, dtype=np.uint64)
    assert np.array_equal(bfv.slot_decode(bfv.slot_encode(v)), v)
    ones = bfv.slot_encode(np.ones(N, dtype=np.uint64))
    assert int(ones[0]) == 1 and np.all(ones[1:] == 0)
    assert np.all(bfv.slot_encode(np.zeros(N, dtype=np.uint64)) == 0)
    prod = core.negacyclic_mul(bfv.slot_encode(v), bfv.slot_encode(w), t) if N <= 1024 else None
    if prod is not None:
        want = (v.astype(object) * w.astype(object)) % t
        assert np.array_equal(bfv.slot_decode(prod), np.array(want, dtype=np.uint64))


def test_exhaustive_toy_codec():
    # S:78 / S:723: toy N=8 context, exhaustive over slot basis vectors and all constants
    t, logN = 17, 3          # 17 = 1 mod 16
    N = 8
    psi = nt.min_primitive_2n_root(t, N)
    for i in range(N):
        e = np.zeros(N, np.uint64); e[i] = 1
        m = core.ntt_inv(e, logN, t, psi)
        for s in range(N):   # the encoded poly evaluates to delta_{is} at slot points
            x = pow(psi, 2 * nt.brev(s, logN) + 1, t)
            assert direct_eval(m, t, x) == (1 if s == i else 0)
    for c in range(t):
        v = np.full(N, c, np.uint64)
        m = core.ntt_inv(v, logN, t, psi)
        assert int(m[0]) == c and np.all(m[1:] == 0)
