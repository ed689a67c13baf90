#!/usr/bin/env python
"""findDmax on the GPU, as Algorithm 1 defines it:

    for i in range(1000):
        D_i = 0
        while evalHEcomputation(N, T, D_i + 1) is correct: D_i += 1
    return average {D_i}

Trial i is one random ct x pt dot product of the real hot path: a batch of B = N/k
plaintext query hypervectors (uniform in +-qmax, SPEC: "probe plaintexts drawn
uniformly at max quantized magnitude") against an encrypted model of uniform class
hypervectors; evalHEcomputation(N, T, D) sums its first D dims
(`ephdc_infer_batch_prefix`) and is correct when the decrypted scores equal the
plaintext dot products mod t (library decryption, `ephdc_decrypt_scores`).  The 1000
trials run as 1000 batches of ONE call per probed D.  The first failing D of each
trial is found by bisection between a correct and a failing D (every probed D is a
real evaluation; a trial still correct at D_cap is reported censored).

Parameters: t = the largest prime = 1 mod 2N below 2^T (the library takes t < 2^30),
T swept over the range where D_max lies between ~1 and D_cap (Fig. "D_max for various
N and log2 t"); q (primes < 2^50, the FP64 kernels):
  * N = 2^11 at the 128-bit-security cap of SPEC.md l.190, Sum log2 q = 54;
  * N = 2^12, 2^13 at the caps (109, 218 bits) D_max is ~2^30 and more for every
    t < 2^30 (the closed form; the run reports these points censored at D_cap), so the
    terminating sweeps there use q = 72 bits (below the cap: more secure, less budget).

usage: python tools/find_dmax.py [--grid default|cap] [--trials 1000] [--dcap 8192]
One JSON line per (N, q, T).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

Q_BITS = {11: (27, 27), 12: (36, 36, 37), 13: (43, 43, 44, 44, 44)}   # SPEC.md l.190 caps: 54 / 109 / 218
GRID = [(11, (27, 27)), (12, (36, 36)), (13, (36, 36))]                  # the terminating sweeps


def predicted_dmax(N: int, t: int, Q: int) -> float:
    """Closed form of tests/test_oracle_noise.py: noise ~ r_t(Q) sqrt(N) t/6 sqrt(D) * 2^1.5."""
    half_delta = (Q // t) / 2
    unit = (Q % t) * math.sqrt(N) * t / 6 * 2 ** 1.5
    return (half_delta / unit) ** 2


class Probe:
    """One (N, T) point: context, key, encrypted uniform model, uniform query HVs."""

    def __init__(self, logN: int, T: int, trials: int, dcap: int, k: int = 2, bits: int = 4, seed: int = 0,
                 device: int = 0, q_bits=None):
        import torch
        import ephdc_inputs as inp
        import paper_2511_00737_b200 as eph
        self.torch, self.eph = torch, eph
        N = 1 << logN
        t = eph.find_ntt_primes(logN, [T])[0]
        q = eph.find_ntt_primes(logN, list(q_bits or Q_BITS[logN]), exclude=[t])
        self.N, self.t, self.q, self.k, self.dcap, self.trials = N, t, q, k, dcap, trials
        self.Q = math.prod(q)
        qmax = (1 << (bits - 1)) - 1
        self.ctx = eph.Context(log2N=logN, q=q, t=t, k=k, D_live=dcap, D_stored=dcap, F=64, feat_unsigned=False,
                               Qbits=bits, Cbits=bits, qshift=0, device=device)
        assert self.ctx.arith == "f64"
        self.B = self.ctx.B
        self.nq = trials * self.B
        rng = np.random.default_rng([seed, logN, T])
        self.C = rng.integers(-qmax, qmax + 1, size=(k, dcap), dtype=np.int8)       # class HVs (host, encrypted)
        self.sk = eph.SecretKey(self.ctx, 1000 + seed)
        self.model = eph.EncryptedModel(self.ctx, self.sk, self.C, 2000 + seed)
        g = torch.Generator(device="cuda")
        g.manual_seed(int(rng.integers(1 << 62)))
        self.H = torch.randint(-qmax, qmax + 1, (dcap, self.nq), generator=g, device="cuda", dtype=torch.int8)
        self.ws = eph.Workspace(self.ctx, self.nq)
        self.Cd = torch.from_numpy(self.C.astype(np.float64)).cuda()

    def expected(self, dims: np.ndarray) -> np.ndarray:
        """Plaintext dot products of every trial's first dims[b] dims, centered mod t: [nq][k]."""
        torch = self.torch
        out = np.empty((self.nq, self.k), dtype=np.int64)
        for b, D in enumerate(dims):
            cols = slice(b * self.B, (b + 1) * self.B)
            s = (self.Cd[:, :D] @ self.H[:D, cols].double()).T        # exact: |s| < 2^53
            out[cols] = s.cpu().numpy().astype(np.int64)
        t = self.t
        return ((out + (t - 1) // 2) % t) - (t - 1) // 2

    def correct(self, dims: np.ndarray) -> np.ndarray:
        """evalHEcomputation(N, T, dims[b]) is correct, per trial b."""
        cts = self.eph.infer_batch_prefix(self.ctx, self.model, self.ws, self.H, self.nq, dims)
        self.torch.cuda.synchronize()
        S, _ = self.eph.decrypt_scores(self.ctx, self.sk, cts.cpu().numpy().view(np.uint64), self.nq)
        ok = (S == self.expected(dims)).reshape(self.trials, self.B * self.k).all(axis=1)
        return ok

    def find_dmax(self):
        """Per trial: bisection between lo (correct; D = 0 sums nothing) and hi (failing)
        until hi = lo + 1 -- D_i = lo decrypts correctly and D_i + 1 does not.  (The
        literal loop stops at the FIRST failing length; with a noise random walk a
        failure can in principle be followed by a correct longer prefix, so bisection
        can land on a later boundary -- tests/test_gpu_find_dmax.py checks D_i and
        D_i + 1 with the oracle.)  Returns (D_i, censored mask, #evaluations)."""
        n = self.trials
        lo = np.zeros(n, dtype=np.int64)                  # D = 0: nothing summed, trivially correct
        hi = np.full(n, self.dcap + 1, dtype=np.int64)
        top = self.correct(np.full(n, self.dcap, dtype=np.uint32))
        lo[top] = self.dcap
        evals = 1
        while np.any(hi - lo > 1):
            mid = np.where(hi - lo > 1, (lo + hi) // 2, lo)
            ok = self.correct(mid.astype(np.uint32))
            act = hi - lo > 1
            lo = np.where(act & ok, mid, lo)
            hi = np.where(act & ~ok, mid, hi)
            evals += 1
        return lo, top, evals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="default", choices=["default", "cap"])
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--dcap", type=int, default=8192)
    a = ap.parse_args()
    import paper_2511_00737_b200 as eph

    if a.grid == "cap":   # N = 2^12, 2^13 at the SPEC caps, the largest t < 2^30: censored at D_cap
        plan = [(12, Q_BITS[12], [29]), (13, Q_BITS[13], [29])]
    else:
        plan = []
        for logN, qb in GRID:
            Ts = []
            for T in range(29, 10, -1):   # predicted D_max from ~1/4 to 2 D_cap
                try:
                    t = eph.find_ntt_primes(logN, [T])[0]
                except eph.EphdcError:      # no prime = 1 mod 2N below 2^T
                    break
                if t.bit_length() != T:
                    continue
                q = eph.find_ntt_primes(logN, list(qb), exclude=[t])
                pd = predicted_dmax(1 << logN, t, math.prod(q))
                if 0.25 <= pd <= 2 * a.dcap:
                    Ts.append(T)
            plan.append((logN, qb, Ts))
    for logN, qb, Ts in plan:
        for T in sorted(Ts, reverse=True):
            t0 = time.perf_counter()
            p = Probe(logN, T, a.trials, a.dcap, q_bits=qb)
            t1 = time.perf_counter()
            Di, cens, evals = p.find_dmax()
            t2 = time.perf_counter()
            print(json.dumps({"N": 1 << logN, "log2_t": T, "t": p.t, "q": p.q, "log2_Q": round(math.log2(p.Q), 2),
                              "trials": a.trials, "batch_B": p.B, "D_cap": a.dcap,
                              "D_max_mean": float(Di.mean()), "D_max_std": float(Di.std()),
                              "D_max_min": int(Di.min()), "D_max_max": int(Di.max()),
                              "censored_trials": int(cens.sum()), "evaluations": evals,
                              "predicted_D_max": round(predicted_dmax(1 << logN, p.t, p.Q), 2),
                              "setup_s": round(t1 - t0, 2), "search_s": round(t2 - t1, 2)}), flush=True)
            del p


if __name__ == "__main__":
    main()
