"""Oracle number theory (plain Python integers) -- TEST INFRASTRUCTURE ONLY.

* NTT-friendly primes: BASELINE.json configs[0..4] ask for primes = 1 (mod 2N),
  "largest below each bound"; SURVEY 8(c) reading #18 makes a chain distinct and
  descending and excludes t.
* psi: a primitive 2N-th root of unity mod p (needed for the negacyclic NTT
  implied by BFV over Z[X]/(X^N+1)).  Reading #2: the MINIMAL one.
* brev: bit reversal, used by the slot order of reading #1.
"""
from __future__ import annotations

from typing import Iterable, List, Sequence

# Deterministic Miller-Rabin witnesses, valid for n < 3.3e24 (covers 64-bit).
_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def largest_ntt_prime_below(bound: int, two_n: int, exclude: Iterable[int] = ()) -> int:
    """Largest prime p < bound with p = 1 (mod two_n), p not in exclude."""
    ex = set(exclude)
    p = ((bound - 2) // two_n) * two_n + 1      # largest value = 1 mod 2N that is < bound
    while p > two_n:
        if p not in ex and is_prime(p):
            return p
        p -= two_n
    raise ValueError("no NTT prime below bound")


def prime_chain(bits: Sequence[int], log2N: int, exclude: Iterable[int] = ()) -> List[int]:
    """One prime per bound 2^bits[i]; distinct; each the largest not yet used."""
    two_n = 2 << log2N
    used = list(exclude)
    out: List[int] = []
    for b in bits:
        p = largest_ntt_prime_below(1 << b, two_n, used)
        out.append(p)
        used.append(p)
    return out


def plaintext_modulus(t_bits: int, log2N: int, t_fixed=None) -> int:
    if t_fixed is not None:
        return t_fixed
    return largest_ntt_prime_below(1 << t_bits, 2 << log2N)


def _small_factors(n: int) -> List[int]:
    f, d = [], 2
    while d * d <= n:
        if n % d == 0:
            f.append(d)
            while n % d == 0:
                n //= d
        d += 1 if d == 2 else 2
    if n > 1:
        f.append(n)
    return f


def any_primitive_2n_root(p: int, two_n: int) -> int:
    """Some x with ord(x) = 2N: x = g^((p-1)/2N) is one iff x^N = -1 (2N a power of 2)."""
    assert (p - 1) % two_n == 0
    e = (p - 1) // two_n
    for g in range(2, p):
        x = pow(g, e, p)
        if pow(x, two_n // 2, p) == p - 1:
            return x
    raise ValueError("no primitive root")


def min_primitive_2n_root(p: int, N: int) -> int:
    """Reading #2: psi = min over all primitive 2N-th roots = min_{k odd} psi0^k."""
    two_n = 2 * N
    psi0 = any_primitive_2n_root(p, two_n)
    best = psi0
    sq = psi0 * psi0 % p
    x = psi0
    for _ in range(N - 1):          # odd powers psi0^1, psi0^3, ..., psi0^(2N-1)
        x = x * sq % p
        if x < best:
            best = x
    return best


def brev(i: int, bits: int) -> int:
    r = 0
    for _ in range(bits):
        r = (r << 1) | (i & 1)
        i >>= 1
    return r


def crt_product(qs: Sequence[int]) -> int:
    Q = 1
    for q in qs:
        Q *= q
    return Q
