"""Seeded synthetic inputs and the configuration table (c1 ... c5).

This module is shared by the product path and by the oracle.  It holds NO
arithmetic of the method (no primes, no NTT, no encoding, no encryption): only
the sizes BASELINE.json fixes and numpy-seeded generators for the raw inputs
(feature matrices, the bipolar projection base, uniform residues for the c5
microbench).  Both sides receive these arrays as inputs.

Recipe:
  * seeds are 2511007370 + config index (c1=1 ... c5=5; c1q3 reuses c1's);
  * clusters: per class a centre mu ~ U[lo, hi] per feature, samples
    x = clip(rint(mu + sigma * N(0,1))) (BASELINE.json configs[0..3]);
  * 64 training samples per class (configs[0] states 64; reading #15 extends
    it to c2..c4); query i belongs to cluster i mod k (reading #17);
  * projection P[d][f] = +1/-1 with probability 1/2, rows d >= D_live are 0
    (configs[0..3] "seeded bipolar +-1 projection").
These inputs stand in for the paper's Face / MNIST / Emotion workloads
(PAPER.md l.717-730); none of those datasets is reproduced.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Tuple

import numpy as np

BASE_SEED = 2511007370


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    index: int                 # 1..5, selects the seed
    log2N: int                 # ring degree N = 2^log2N
    t_bits: int                # t = largest prime < 2^t_bits, t = 1 mod 2N (unless t_fixed)
    t_fixed: Optional[int]     # c1: t = 65537 exactly
    q_bits: Tuple[int, ...]    # one bound per RNS prime, in order
    k: int                     # classes
    F: int                     # features
    feat_unsigned: bool        # uint8 (c3) vs int8 features
    D_live: int
    D_stored: int
    Cbits: int                 # class HV bits (BASELINE.json)
    nq: int                    # queries per step
    mu_lo: int
    mu_hi: int
    sigma: float
    n_train_per_class: int = 64
    sigma_e: float = 3.2       # BFV error std-dev (configs[0])

    @property
    def N(self) -> int:
        return 1 << self.log2N

    @property
    def L(self) -> int:
        return len(self.q_bits)

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index


CONFIGS: Dict[str, Config] = {
    # BASELINE.json configs[0] literally: one 30-bit q (noise-infeasible)
    "c1": Config("c1", 1, 10, 17, 65537, (30,), 2, 64, False, 1024, 1024, 4, 16,
                 -40, 40, 12.0),
    # c1 with 3 x 30-bit primes: the decryptable toy variant (reading #22)
    "c1q3": Config("c1q3", 1, 10, 17, 65537, (30, 30, 30), 2, 64, False, 1024, 1024, 4, 16,
                   -40, 40, 12.0),
    # configs[1]
    "c2": Config("c2", 2, 12, 20, None, (36, 36, 37), 2, 608, False, 4096, 4096, 4, 1024,
                 -40, 40, 12.0),
    # configs[2]
    "c3": Config("c3", 3, 13, 22, None, (43, 43, 44, 44, 44), 10, 784, True, 8192, 8192, 4, 8192,
                 0, 255, 30.0),
    # configs[3]
    "c4": Config("c4", 4, 14, 30, None, (48,) * 9, 7, 1024, False, 10000, 16384, 8, 65536,
                 -40, 40, 12.0),
}

# configs[4]: kernel microbench sweep (standalone NTT / MAC on uniform residues)
C5_LOG2N = (12, 13, 14, 15, 16)
C5_L = (1, 3, 5, 9, 16)
C5_WORD_BITS = (30, 60)
C5_BATCHES = (1, 16, 256, 4096, 65536)
C5_WORKING_SET_CAP = 32 << 30


def _clip_range(cfg: Config) -> Tuple[int, int]:
    return (0, 255) if cfg.feat_unsigned else (-128, 127)


def gen_features(cfg: Config, nq: Optional[int] = None, stream: int = 0):
    """Returns (X_train, y_train, X_query, y_query).

    X_* are uint8 (c3) or int8 row-major [n, F]; y_* int64 class labels.
    Query i is drawn from cluster i mod k.  stream > 0 draws an independent query set
    (seed (cfg.seed, stream)) from the same clusters and training set: the per-rank
    query streams of a multi-GPU run.
    """
    nq = cfg.nq if nq is None else nq
    rng = np.random.default_rng(cfg.seed)
    mu = rng.uniform(cfg.mu_lo, cfg.mu_hi, size=(cfg.k, cfg.F))
    lo, hi = _clip_range(cfg)
    dt = np.uint8 if cfg.feat_unsigned else np.int8

    def draw(labels: np.ndarray, g) -> np.ndarray:
        z = g.standard_normal(size=(labels.size, cfg.F))
        x = np.clip(np.rint(mu[labels] + cfg.sigma * z), lo, hi)
        return x.astype(dt)

    y_train = np.repeat(np.arange(cfg.k, dtype=np.int64), cfg.n_train_per_class)
    X_train = draw(y_train, rng)
    y_query = np.arange(nq, dtype=np.int64) % cfg.k
    X_query = draw(y_query, rng if stream == 0 else np.random.default_rng([cfg.seed, stream]))
    return X_train, y_train, X_query, y_query


def gen_projection(cfg: Config) -> np.ndarray:
    """Bipolar base P [D_stored, F] int8 in {+1,-1}; rows >= D_live are 0."""
    rng = np.random.default_rng(cfg.seed + 1000)
    bits = rng.integers(0, 2, size=(cfg.D_live, cfg.F), dtype=np.int8)
    P = np.zeros((cfg.D_stored, cfg.F), dtype=np.int8)
    P[: cfg.D_live] = (2 * bits - 1).astype(np.int8)
    return P


def gen_residues(moduli: List[int], n_poly: int, N: int, seed: int) -> np.ndarray:
    """Uniform residues, shape [n_poly, L, N] uint64, entry [., j, .] < moduli[j]."""
    rng = np.random.default_rng(seed)
    out = np.empty((n_poly, len(moduli), N), dtype=np.uint64)
    for j, q in enumerate(moduli):
        out[:, j, :] = rng.integers(0, q, size=(n_poly, N), dtype=np.uint64)
    return out


def c5_max_batch(log2N: int, L: int, word_bytes: int = 8) -> int:
    """Largest MAC term count D whose ct+pt+out working set fits the 32 GB cap."""
    N = 1 << log2N
    per_term = 3 * L * N * word_bytes          # 2 ciphertext polys + 1 plaintext poly
    return max(1, (C5_WORKING_SET_CAP - 2 * L * N * word_bytes) // per_term)


# c5 sweep (BASELINE.json configs[4]): word classes -- 30-bit primes (u64 words; u32
# words through the *32 entry points), 48-bit (the FP64 kernels' range) and 60-bit
# primes -- for every N and L; batches 1 ... 65536 capped by the 32 GB working set.
C5_PRIME_BITS = (30, 48, 60)


def c5_points(kind: str = "all"):
    """[(log2N, L, bits, word_bytes, [batches])] of the c5 sweep.  kind: "all" (every
    N x L x word class, batches C5_BATCHES capped at the working set) or "quick"."""
    pts = []
    if kind == "quick":
        grid = [(lg, L, b, 8) for lg in C5_LOG2N for L, b in ((9, 48), (5, 60), (16, 30))]
    else:
        grid = [(lg, L, b, 8) for lg in C5_LOG2N for L in C5_L for b in C5_PRIME_BITS]
        grid += [(lg, L, 30, 4) for lg in C5_LOG2N for L in C5_L]
    for lg, L, b, wb in grid:
        cap = max(1, C5_WORKING_SET_CAP // (L * (1 << lg) * wb))
        bs = sorted({min(x, cap) for x in C5_BATCHES})
        pts.append((lg, L, b, wb, bs))
    return pts


def c5_residues_torch(moduli: List[int], n_poly: int, N: int, seed: int, device, dtype=None):
    """Uniform residues [n_poly, L, N] (int64, or the given torch dtype) generated ON the
    device with torch's seeded Philox generator: the bulk inputs of the c5 sweep (too
    large for numpy); tests copy the sampled polynomials they check back to the host."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((n_poly, len(moduli), N), dtype=torch.int64, device=device)
    for j, q in enumerate(moduli):
        out[:, j, :] = torch.randint(0, int(q), (n_poly, N), generator=g, device=device, dtype=torch.int64)
    return out if dtype is None else out.to(dtype)
