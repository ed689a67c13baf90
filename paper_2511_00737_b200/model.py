"""Server-side model build (CS1, untimed, once): training samples are projected on
the GPU (ephdc_encode_raw), then bundled and quantised on the host.

* single-pass training: class HV = sum of the class's encoded samples;
* class quantisation to C bits (reading #14): per class, round-half-away
  of v * cmax / max|v|;
* query width Q (reading #12): largest Q <= 8 with D_live * qmax * cmax <= (t-1)/2,
  so that no score wraps mod t;
* query shift s (reading #13): smallest s with max|acc_train| <= qmax * 2^s.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def query_bits(D_live: int, Cbits: int, t: int) -> int:
    cmax = (1 << (Cbits - 1)) - 1
    limit = (t - 1) // 2
    Q = 8
    while Q >= 2 and D_live * ((1 << (Q - 1)) - 1) * cmax > limit:
        Q -= 1
    if Q < 2:
        raise ValueError("no query width keeps the scores below t/2")
    return Q


def query_shift(acc_train: np.ndarray, Qbits: int) -> int:
    peak = int(np.max(np.abs(acc_train)))
    qmax = (1 << (Qbits - 1)) - 1
    s = 0
    while (qmax << s) < peak:
        s += 1
    return s


def bundle_and_quantise(acc_train: np.ndarray, y_train: np.ndarray, k: int, Cbits: int) -> np.ndarray:
    """acc_train int32/int64 [D, n]; returns class HVs int8 [k, D]."""
    cmax = (1 << (Cbits - 1)) - 1
    onehot = np.zeros((acc_train.shape[1], k), dtype=np.int64)
    onehot[np.arange(acc_train.shape[1]), y_train] = 1
    v = (acc_train.astype(np.int64) @ onehot).T               # [k, D] class sums
    mag = np.abs(v)
    M = mag.max(axis=1, keepdims=True)
    safe = np.where(M == 0, 1, M)
    r = (2 * mag * cmax + safe) // (2 * safe)                 # round half away from zero
    r = np.where(M == 0, 0, r)
    return (np.sign(v) * r).astype(np.int8)


def train(acc_train: np.ndarray, y_train: np.ndarray, k: int, Cbits: int, Qbits: int) -> Tuple[np.ndarray, int]:
    return bundle_and_quantise(acc_train, y_train, k, Cbits), query_shift(acc_train, Qbits)
