"""Oracle end-to-end driver for one configuration -- TEST INFRASTRUCTURE ONLY.

Server setup (CS1): encode training samples, calibrate the query shift, bundle
(P:120-122), quantise classes to C bits, keygen, encrypt.
Client (CS2): encode + quantise queries, per batch sum_d CT_d (.) PT_{b,d}.
Server decide (CS3): decrypt, decode, argmax.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

import ephdc_inputs as inp
from . import hdc
from .bfv import OracleBFV

SK_SEED_OFFSET = 17
ENC_SEED_OFFSET = 29


@dataclasses.dataclass
class OracleModel:
    cfg: inp.Config
    bfv: OracleBFV
    Qbits: int
    qshift: int
    class_hv: np.ndarray        # int8 [k, D_live]
    sk_seed: int
    enc_seed: int


def build_model(cfg: inp.Config, P: np.ndarray, X_train: np.ndarray, y_train: np.ndarray) -> OracleModel:
    bfv = OracleBFV(cfg)
    Qbits = hdc.choose_Qbits(cfg.D_live, cfg.Cbits, bfv.t)
    acc_train = hdc.encode_raw(P, X_train, cfg.D_live)
    s = hdc.calibrate_shift(acc_train, Qbits)
    v = hdc.bundle(acc_train, y_train, cfg.k)
    C = hdc.quantise_classes(v, cfg.Cbits)
    sk_seed = cfg.seed + SK_SEED_OFFSET
    enc_seed = cfg.seed + ENC_SEED_OFFSET
    bfv.keygen(sk_seed)
    return OracleModel(cfg, bfv, Qbits, s, C, sk_seed, enc_seed)


def encode_queries(m: OracleModel, P: np.ndarray, X: np.ndarray) -> np.ndarray:
    """H [D_live, nq] int8 (dim-major)."""
    acc = hdc.encode_raw(P, X, m.cfg.D_live)
    return hdc.quantise_queries(acc, m.qshift, m.Qbits)


def infer_all(m: OracleModel, H: np.ndarray, model: Optional[np.ndarray] = None) -> np.ndarray:
    nq = H.shape[1]
    nb = m.bfv.n_batches(nq)
    out = np.empty((nb, 2, m.bfv.L, m.bfv.N), dtype=np.uint64)
    for b in range(nb):
        out[b] = m.bfv.infer_batch(H, nq, b, model=model, class_hv=m.class_hv, enc_seed=m.enc_seed)
    return out
