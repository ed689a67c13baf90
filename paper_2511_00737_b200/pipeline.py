"""Config-level setup of the product path: parameters, model build, keys, encrypted model.

Used by bench.py, __graft_entry__.smoke() and the GPU tests.  Primes and psi come
from the library (ephdc_find_ntt_primes / ctx_create), the model build from
ephdc_query_bits / ephdc_train_model (host C++), every device step from libephdc
kernels; this module only sequences the calls.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

import ephdc_inputs as inp
from . import Context, EncryptedModel, SecretKey, encode_raw, find_ntt_primes, query_bits, train_model

SK_SEED_OFFSET = 17      # deterministic test keys: the oracle driver's seed schedule (inputs, not arithmetic)
ENC_SEED_OFFSET = 29


@dataclasses.dataclass
class Setup:
    cfg: inp.Config
    ctx: Context
    sk: SecretKey
    model: EncryptedModel
    class_hv: np.ndarray
    P_dev: object          # torch cuda [D_stored, F] int8
    Qbits: int
    qshift: int


def primes_for(cfg: inp.Config):
    if cfg.t_fixed is not None:
        t = cfg.t_fixed
    else:
        t = find_ntt_primes(cfg.log2N, [cfg.t_bits])[0]
    q = find_ntt_primes(cfg.log2N, list(cfg.q_bits), exclude=[t])
    return t, q


def make_context(cfg: inp.Config, t: int, q, Qbits: int, qshift: int, device: int = 0, arith: int = 0,
                 encoder: int = 0) -> Context:
    return Context(log2N=cfg.log2N, q=q, t=t, k=cfg.k, D_live=cfg.D_live, D_stored=cfg.D_stored, F=cfg.F,
                   feat_unsigned=cfg.feat_unsigned, Qbits=Qbits, Cbits=cfg.Cbits, qshift=qshift,
                   sigma_e=cfg.sigma_e, device=device, arith=arith, encoder=encoder)


def build(cfg: inp.Config, P: np.ndarray, X_train: np.ndarray, y_train: np.ndarray, device: int = 0,
          sk_seed: Optional[int] = None, enc_seed: Optional[int] = None, arith: int = 0,
          encoder: int = 0, deterministic: bool = False) -> Setup:
    """arith: 0 auto (FP64 pipe when eligible), 1 integer pipe, 2 FP64 pipe (ephdc_params.arith);
    encoder: 0 auto (tcgen05 tensor cores), 1 dp4a CUDA cores (ephdc_params.encoder).
    Keys (reading #7): by default the secret key and the model encryption each draw a
    fresh OS key; deterministic=True (parity tests, benchmarks) uses the guessable test
    keys cfg.seed + 17 / + 29 -- the oracle driver's schedule -- unless sk_seed / enc_seed
    name others."""
    import torch
    dev = torch.device("cuda", device)
    t, q = primes_for(cfg)
    Qbits = query_bits(cfg.D_live, cfg.Cbits, t)
    P_dev = torch.from_numpy(np.ascontiguousarray(P)).to(dev)
    # training projection on the GPU (the quantisation fields are unused by encode_raw)
    ctx0 = make_context(cfg, t, q, Qbits, 0, device, arith, encoder)
    Xt = torch.from_numpy(np.ascontiguousarray(X_train).view(np.int8)).to(dev)
    acc = encode_raw(ctx0, Xt, P_dev).cpu().numpy()
    torch.cuda.synchronize(dev)
    class_hv, qshift = train_model(acc, y_train, cfg.k, cfg.Cbits, Qbits)
    ctx0.close()
    ctx = make_context(cfg, t, q, Qbits, qshift, device, arith, encoder)
    if deterministic:
        sk_seed = cfg.seed + SK_SEED_OFFSET if sk_seed is None else sk_seed
        enc_seed = cfg.seed + ENC_SEED_OFFSET if enc_seed is None else enc_seed
    sk = SecretKey(ctx, sk_seed)
    model = EncryptedModel(ctx, sk, class_hv, enc_seed)
    return Setup(cfg, ctx, sk, model, class_hv, P_dev, Qbits, qshift)
