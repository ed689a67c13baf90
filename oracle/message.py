"""Oracle of the scores message (client -> server) --
TEST INFRASTRUCTURE ONLY.

The message is our serialisation of the nb scores ciphertexts: the residues of prime j
written at b_j = bit_length(q_j) bits each, least significant bit first, one bit
stream over blocks in [nb][2][L] order (include/ephdc.h "scores message").  Written
as the plain definition: one Python integer per value, bit by bit.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np


def message_bytes(nb: int, N: int, q: Sequence[int]) -> int:
    return nb * 2 * N * sum(int(p).bit_length() for p in q) // 8


def pack(ct: np.ndarray, q: Sequence[int]) -> bytes:
    nb, two, L, N = ct.shape
    bits = [int(p).bit_length() for p in q]
    out = bytearray(message_bytes(nb, N, q))
    pos = 0
    for b in range(nb):
        for c in range(two):
            for j in range(L):
                for v in ct[b, c, j].tolist():
                    for k in range(bits[j]):
                        if (v >> k) & 1:
                            out[pos >> 3] |= 1 << (pos & 7)
                        pos += 1
    return bytes(out)


def unpack(msg: bytes, nb: int, N: int, q: Sequence[int]) -> np.ndarray:
    L = len(q)
    bits = [int(p).bit_length() for p in q]
    out = np.zeros((nb, 2, L, N), dtype=np.uint64)
    pos = 0
    for b in range(nb):
        for c in range(2):
            for j in range(L):
                vals = []
                for _ in range(N):
                    v = 0
                    for k in range(bits[j]):
                        v |= ((msg[pos >> 3] >> (pos & 7)) & 1) << k
                        pos += 1
                    vals.append(v)
                out[b, c, j] = np.array(vals, dtype=np.uint64)
    return out
