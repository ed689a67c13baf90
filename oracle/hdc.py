"""Oracle HDC encoder, training and quantisation (numpy) -- TEST INFRASTRUCTURE ONLY.

* encoding: random projection, H = P . x ("multiplying a random base
  hypervector"; BASELINE.json subsystem (a): int8 x bipolar, int32 accumulation).
  Computed as a float64 matmul: every product and partial sum is an integer of
  magnitude < 2^53 (|acc| <= F*255 < 2^18), so the result is exact.
* query quantisation to Q bits (readings #12, #13):
  h = clamp(floor((acc + 2^(s-1)) / 2^s), -qmax, qmax), qmax = 2^(Q-1) - 1.
* shift calibration s: smallest s >= 0 with max|acc_train| <= qmax * 2^s (reading #13).
* single-pass training: class HV = sum of the class's encoded samples.
* class quantisation to C bits (reading #14): per-class max-abs rounding,
  round half away from zero, C_c[d] = sign(v)*floor((2|v|cmax + M)/(2M)).
* similarity = dot product, argmax with lowest index on ties.
"""
from __future__ import annotations

import numpy as np


def encode_raw(P: np.ndarray, X: np.ndarray, D_live: int) -> np.ndarray:
    """acc[d][q] = sum_f P[d][f] * X[q][f] for d < D_live; int64 [D_live, nq]."""
    Pf = P[:D_live].astype(np.float64)
    Xf = X.astype(np.float64)
    acc = Pf @ Xf.T
    out = acc.astype(np.int64)
    assert np.array_equal(out.astype(np.float64), acc)
    return out


def qmax_of(bits: int) -> int:
    return (1 << (bits - 1)) - 1


def choose_Qbits(D_live: int, Cbits: int, t: int, cap: int = 8) -> int:
    """Reading #12: the largest Q with D_live*qmax(Q)*cmax <= (t-1)/2, capped at 8."""
    cmax = qmax_of(Cbits)
    best = None
    for Q in range(2, cap + 1):
        if D_live * qmax_of(Q) * cmax <= (t - 1) // 2:
            best = Q
    if best is None:
        raise ValueError("no query width avoids wrap-around")
    return best


def calibrate_shift(acc_train: np.ndarray, Qbits: int) -> int:
    m = int(np.abs(acc_train).max())
    qm = qmax_of(Qbits)
    s = 0
    while m > qm * (1 << s):
        s += 1
    return s


def quantise_queries(acc: np.ndarray, s: int, Qbits: int) -> np.ndarray:
    qm = qmax_of(Qbits)
    if s == 0:
        h = acc.copy()
    else:
        h = np.floor_divide(acc + (1 << (s - 1)), 1 << s)
    return np.clip(h, -qm, qm).astype(np.int8)


def bundle(acc_train: np.ndarray, y_train: np.ndarray, k: int) -> np.ndarray:
    """v_c = sum over training samples of class c of their (unquantised) HVs, int64 [k, D]."""
    D = acc_train.shape[0]
    v = np.zeros((k, D), dtype=np.int64)
    for c in range(k):
        v[c] = acc_train[:, y_train == c].sum(axis=1)
    return v


def quantise_classes(v: np.ndarray, Cbits: int) -> np.ndarray:
    cmax = qmax_of(Cbits)
    out = np.zeros(v.shape, dtype=np.int8)
    for c in range(v.shape[0]):
        M = int(np.abs(v[c]).max())
        if M == 0:
            continue
        a = np.abs(v[c])
        r = (2 * a * cmax + M) // (2 * M)
        out[c] = (np.sign(v[c]) * r).astype(np.int8)
    return out


def scores(H: np.ndarray, C: np.ndarray) -> np.ndarray:
    """Brute-force integer dot products: score[q][c] = sum_d h[d][q] * C[c][d]; int64 [nq, k]."""
    return H.astype(np.int64).T @ C.astype(np.int64).T


def argmax_lowest(S: np.ndarray) -> np.ndarray:
    return np.argmax(S, axis=1).astype(np.int64)   # numpy returns the first maximum
