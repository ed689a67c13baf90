"""Oracle BFV pipeline of EP-HDC's client-side inference -- TEST INFRASTRUCTURE ONLY.

Parameters (BASELINE.json configs; SURVEY 8(c) readings):
  t, q_j       -- largest primes = 1 mod 2N below the configured bounds (#18)
  psi_t, psi_j -- minimal primitive 2N-th roots (#2)
  Delta        -- floor(Q/t) (#4), Q = prod q_j
  B            -- floor(N/k) queries per ciphertext
Keys / encryption: secret-key BFV (#5), ternary s (#9), uniform a
sampled in the NTT domain (#6, #8), CDT discrete Gaussian e with sigma = 3.2
(BASELINE.json configs[0]; #10).  Decryption: m = round(t*x/Q) mod t, then
slots = NTT_t(m) (CS3; #20), done with Python big integers.
"""
from __future__ import annotations

import ctypes
import math
from decimal import Decimal, getcontext
from typing import List, Optional, Tuple

import numpy as np

from ephdc_inputs import Config
from . import core, hdc, nt

CDT_LEN = 20          # magnitudes 0..19 (6-sigma cut at sigma = 3.2)


def gaussian_cdt(sigma: float = 3.2, n: int = CDT_LEN) -> np.ndarray:
    """Reading #10: cumulative thresholds T[k] = round(2^40 * cdf(k)) * 2^23, T[n-1] = 2^63.

    p(0) = rho(0)/Z, p(k) = 2 rho(k)/Z (k >= 1), rho(x) = exp(-x^2 / (2 sigma^2)),
    Z = rho(0) + 2 sum_{k=1}^{n-1} rho(k).  Evaluated with 50-digit decimals.
    """
    getcontext().prec = 50
    s = Decimal(repr(sigma))
    rho = [(-(Decimal(k) ** 2) / (2 * s * s)).exp() for k in range(n)]
    w = [rho[0]] + [2 * r for r in rho[1:]]
    Z = sum(w)
    out, acc = [], Decimal(0)
    for k in range(n):
        acc += w[k]
        v = acc / Z * (Decimal(2) ** 40)
        out.append(int(v.to_integral_value(rounding="ROUND_HALF_EVEN")) << 23)
    out[-1] = 1 << 63
    return np.array(out, dtype=np.uint64)


class OracleBFV:
    def __init__(self, cfg: Config):
        self.cfg = cfg
        self.logN = cfg.log2N
        self.N = cfg.N
        self.k = cfg.k
        self.t = nt.plaintext_modulus(cfg.t_bits, cfg.log2N, cfg.t_fixed)
        self.q = nt.prime_chain(cfg.q_bits, cfg.log2N, exclude=[self.t])
        self.L = len(self.q)
        self.Q = nt.crt_product(self.q)
        self.psi_t = nt.min_primitive_2n_root(self.t, self.N)
        self.psi = [nt.min_primitive_2n_root(p, self.N) for p in self.q]
        self.delta_big = self.Q // self.t
        self.delta = [self.delta_big % p for p in self.q]
        self.B = self.N // self.k
        self.D_live = cfg.D_live
        self.cdt = gaussian_cdt(cfg.sigma_e)
        self.s = None
        self.s_hat = None
        self._keep = []

    # -- sizes ---------------------------------------------------------------------
    def n_batches(self, nq: int) -> int:
        return (nq + self.B - 1) // self.B

    # -- keys ----------------------------------------------------------------------
    def keygen(self, seed: int) -> np.ndarray:
        s = np.empty(self.N, dtype=np.int8)
        core.lib().or_sample_ternary(seed, self.N, core.ptr(s))
        self.s = s
        sh = np.empty((self.L, self.N), dtype=np.uint64)
        for j, p in enumerate(self.q):
            sh[j] = np.where(s < 0, p - 1, s.astype(np.int64)).astype(np.uint64)
        for j, p in enumerate(self.q):
            sh[j] = core.ntt_fwd(sh[j], self.logN, p, self.psi[j])
        self.s_hat = np.ascontiguousarray(sh)
        return s

    def _struct(self, enc_seed: int = 0) -> core.OrBfv:
        q = core.u64arr(self.q)
        psi = core.u64arr(self.psi)
        delta = core.u64arr(self.delta)
        sh = self.s_hat if self.s_hat is not None else np.zeros((self.L, self.N), np.uint64)
        cdt = np.ascontiguousarray(self.cdt)
        self._keep = [q, psi, delta, sh, cdt]
        return core.OrBfv(self.logN, self.L, core.ptr(q), core.ptr(psi), self.t, self.psi_t,
                          self.k, self.D_live, core.ptr(delta), core.ptr(sh), enc_seed,
                          core.ptr(cdt), len(cdt))

    # -- slot codec (reading #1) ---------------------------------------------
    def slot_encode(self, v: np.ndarray) -> np.ndarray:
        return core.ntt_inv(np.asarray(v, dtype=np.uint64) % np.uint64(self.t), self.logN, self.t, self.psi_t)

    def slot_decode(self, m: np.ndarray) -> np.ndarray:
        return core.ntt_fwd(m, self.logN, self.t, self.psi_t)

    # -- server: encrypt the model ------------------------------------------------
    def encrypt_dims(self, class_hv: np.ndarray, enc_seed: int, d0: int, nd: int) -> np.ndarray:
        assert self.s_hat is not None
        C = np.ascontiguousarray(class_hv, dtype=np.int8)
        out = np.empty((nd, self.L, 2, self.N), dtype=np.uint64)
        st = self._struct(enc_seed)
        core.lib().or_encrypt_dims(ctypes.byref(st), core.ptr(C), d0, nd, core.ptr(out))
        return out

    # -- client ----------------------------------------------------------------------
    def plaintext_ntts(self, H: np.ndarray, nq: int, b: int, d0: int, nd: int) -> np.ndarray:
        Hc = np.ascontiguousarray(H, dtype=np.int8)
        out = np.empty((nd, self.L, self.N), dtype=np.uint64)
        st = self._struct()
        core.lib().or_plaintext_ntts(ctypes.byref(st), core.ptr(Hc), nq, b, d0, nd, core.ptr(out))
        return out

    def infer_batch(self, H: np.ndarray, nq: int, b: int, model: Optional[np.ndarray] = None,
                    class_hv: Optional[np.ndarray] = None, enc_seed: int = 0,
                    counters: Optional[np.ndarray] = None) -> np.ndarray:
        """Scores ciphertext of batch b: [2][L][N] canonical NTT form."""
        Hc = np.ascontiguousarray(H, dtype=np.int8)
        acc = np.empty((2, self.L, self.N), dtype=np.uint64)
        st = self._struct(enc_seed)
        m = None if model is None else np.ascontiguousarray(model, dtype=np.uint64)
        C = None if class_hv is None else np.ascontiguousarray(class_hv, dtype=np.int8)
        cnt = np.zeros(3, dtype=np.uint64) if counters is None else counters
        core.lib().or_infer_batch(ctypes.byref(st), core.ptr(Hc), nq, b, core.ptr(m), core.ptr(C),
                                  core.ptr(acc), core.ptr(cnt))
        return acc

    def infer_batch_scaled(self, H: np.ndarray, nq: int, b: int, g: int, scales, model: Optional[np.ndarray] = None,
                           class_hv: Optional[np.ndarray] = None, enc_seed: int = 0,
                           counters: Optional[dict] = None) -> np.ndarray:
        """Client evaluation with the accumulator scaling of PAPER.md l.429-431 ("a scaling
        operation ... after every g HE additions", g = 512): the dims are accumulated in
        ascending groups of g and after group j the running accumulator is multiplied by
        the plaintext constant s_j^-1 mod t (mul_cp(acc, s_j^-1) after each
        group, ceil(D/g) scaling multiplies).  A plaintext constant c is the constant
        polynomial c (slot encoding of an all-c vector); in the NTT domain of q_j
        the product is the pointwise product with lift_j(c) (centered lift, reading #3)
        -- written here as that literal sequence, Python integers for the products."""
        D = self.D_live
        groups = [(d0, min(D, d0 + g)) for d0 in range(0, D, g)]
        if len(scales) != len(groups):
            raise ValueError("one scale per group of g dims")
        acc = [[[0] * self.N for _ in range(self.L)] for _ in range(2)]
        Hc = np.ascontiguousarray(H, dtype=np.int8)
        m = None if model is None else np.ascontiguousarray(model, dtype=np.uint64)
        C = None if class_hv is None else np.ascontiguousarray(class_hv, dtype=np.int8)
        n_mul = n_add = n_scale = 0
        for (d0, d1), s in zip(groups, scales):
            if s % self.t == 0:
                raise ValueError("scale must be invertible mod t")
            part = np.empty((2, self.L, self.N), dtype=np.uint64)
            cnt = np.zeros(3, dtype=np.uint64)
            st = self._struct(enc_seed)
            core.lib().or_infer_batch_range(ctypes.byref(st), core.ptr(Hc), nq, b, d0, d1, core.ptr(m), core.ptr(C),
                                            core.ptr(part), core.ptr(cnt))
            n_mul += int(cnt[0])
            n_add += int(cnt[1]) + (1 if d0 > 0 else 0)      # folding the group into the accumulator
            sinv = pow(int(s), -1, self.t)
            lifted = sinv if sinv <= (self.t - 1) // 2 else sinv - self.t
            for c in range(2):
                for j, p in enumerate(self.q):
                    f = lifted % p
                    pj = part[c, j].tolist()
                    acc[c][j] = [((a + x) * f) % p for a, x in zip(acc[c][j], pj)]
            n_scale += 1
        if counters is not None:
            counters.update(mul_cp=n_mul, add_cc=n_add, scale=n_scale, rot=0)
        return np.array(acc, dtype=np.uint64)

    # -- HE-HDC-SR, the server-side SIMD baseline -----------
    def sr_encrypt_queries(self, H: np.ndarray, nq: int, b: int, enc_seed: int) -> np.ndarray:
        """Client: batch b's query hypervectors as D_live ciphertexts [D][L][2][N]."""
        Hc = np.ascontiguousarray(H, dtype=np.int8)
        out = np.empty((self.D_live, self.L, 2, self.N), dtype=np.uint64)
        st = self._struct(enc_seed)
        core.lib().or_encrypt_queries(ctypes.byref(st), core.ptr(Hc), nq, b, 0, self.D_live, core.ptr(out))
        return out

    def sr_server_eval(self, class_hv: np.ndarray, qct: np.ndarray) -> np.ndarray:
        """Server: sum_d qct_d (.) encode(tile_d) with the plaintext class tiles -> [2][L][N]."""
        C = np.ascontiguousarray(class_hv, dtype=np.int8)
        q = np.ascontiguousarray(qct, dtype=np.uint64)
        acc = np.empty((2, self.L, self.N), dtype=np.uint64)
        st = self._struct()
        core.lib().or_server_eval(ctypes.byref(st), core.ptr(C), core.ptr(q), core.ptr(acc))
        return acc

    # -- server: decrypt / decode (CS3) ------------------------------------------
    def decrypt_poly(self, ct: np.ndarray) -> List[int]:
        """Phase x = c0 + c1*s in coefficient form, CRT-combined into [0, Q) (Python ints)."""
        ctc = np.ascontiguousarray(ct, dtype=np.uint64).reshape(2, self.L, self.N)
        ph = np.empty((self.L, self.N), dtype=np.uint64)
        st = self._struct()
        core.lib().or_decrypt_phase(ctypes.byref(st), core.ptr(ctc), core.ptr(ph))
        Q = self.Q
        coef = []
        for p in self.q:
            Mj = Q // p
            coef.append(Mj * pow(Mj, -1, p))
        cols = [ph[j].tolist() for j in range(self.L)]
        x = [sum(cols[j][i] * coef[j] for j in range(self.L)) % Q for i in range(self.N)]
        return x

    def decrypt(self, ct: np.ndarray) -> np.ndarray:
        """Slot values in [0, t): m = floor((t*x + floor(Q/2)) / Q) mod t, slots = NTT_t(m)."""
        x = self.decrypt_poly(ct)
        Q, t = self.Q, self.t
        m = np.array([((t * xi + Q // 2) // Q) % t for xi in x], dtype=np.uint64)
        return self.slot_decode(m)

    def noise_max(self, ct: np.ndarray, slots_expected: np.ndarray) -> int:
        """Infinity norm of x - Delta*m_expected (centered mod Q), an exact Python int."""
        x = self.decrypt_poly(ct)
        m = self.slot_encode(np.asarray(slots_expected, dtype=np.int64) % self.t).tolist()
        Q, dl = self.Q, self.delta_big
        worst = 0
        for xi, mi in zip(x, m):
            r = (xi - dl * int(mi)) % Q
            if r > Q // 2:
                r -= Q
            worst = max(worst, abs(r))
        return worst

    def noise_bits(self, ct: np.ndarray, slots_expected: np.ndarray) -> float:
        """log2 of the infinity norm of x - Delta*m_expected (centered mod Q)."""
        worst = self.noise_max(ct, slots_expected)
        return math.log2(worst) if worst else 0.0      # worst can exceed 2^64 (Python int)

    def decode_scores(self, cts: np.ndarray, nq: int) -> Tuple[np.ndarray, np.ndarray]:
        """cts [nb][2][L][N] -> centered scores [nq, k] int64 and argmax labels [nq]."""
        S = np.zeros((nq, self.k), dtype=np.int64)
        t = self.t
        for b in range(self.n_batches(nq)):
            v = self.decrypt(cts[b]).astype(np.int64)
            v = np.where(v > (t - 1) // 2, v - t, v)
            nb = min(self.B, nq - b * self.B)
            S[b * self.B: b * self.B + nb] = v[: self.k * nb].reshape(nb, self.k)
        return S, hdc.argmax_lowest(S)
