"""ctypes binding of libephdc.so: argument marshalling only, same names as include/ephdc.h.

Every compute step runs inside the library's CUDA kernels.  If the library is
missing this module raises at import time -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libephdc.so")

MAX_PRIMES = 16

c_u64 = ctypes.c_uint64
c_u32 = ctypes.c_uint32
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_st = ctypes.c_int  # ephdc_status


class EphdcError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed: status {status} ({msg})")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [
        ("log2N", c_u32), ("L", c_u32), ("q", ctypes.POINTER(c_u64)), ("t", c_u64),
        ("k", c_u32), ("D_live", c_u32), ("D_stored", c_u32), ("F", c_u32),
        ("feat_unsigned", c_u32), ("Qbits", c_u32), ("Cbits", c_u32), ("qshift", c_u32),
        ("sigma_e", ctypes.c_double), ("arith", c_u32), ("encoder", c_u32),
    ]


ARITH_AUTO, ARITH_INT, ARITH_F64 = 0, 1, 2


class Seed(ctypes.Structure):
    """ephdc_seed: 256-bit ChaCha20 key of the random streams (reading #7)."""
    _fields_ = [("key", c_u32 * 8)]


class Plan(ctypes.Structure):
    _fields_ = [("flags", c_u32), ("bg", c_u32), ("G", c_u32), ("m_batches", c_u32)]


class CtxInfo(ctypes.Structure):
    _fields_ = [
        ("N", c_u32), ("L", c_u32), ("B", c_u32), ("k", c_u32),
        ("t", c_u64), ("psi_t", c_u64),
        ("q", c_u64 * MAX_PRIMES), ("psi", c_u64 * MAX_PRIMES), ("delta", c_u64 * MAX_PRIMES),
        ("fused_split", c_u32), ("fused_chunks", c_u32), ("device", c_int),
        ("arith", c_u32), ("f64_red_every", c_u32),
    ]


_SIGS = {
    "ephdc_status_string": (ctypes.c_char_p, [c_st]),
    "ephdc_abi_version": (c_int, []),
    "ephdc_find_ntt_primes": (c_st, [c_u32, c_vp, c_u32, c_vp, c_u32, c_vp]),
    "ephdc_min_psi": (c_st, [c_u64, c_u32, c_vp]),
    "ephdc_gaussian_cdt": (c_st, [ctypes.c_double, c_vp]),
    "ephdc_launch_count": (c_u64, []),
    "ephdc_query_bits": (c_st, [c_u32, c_u32, c_u64, c_vp]),
    "ephdc_train_model": (c_st, [c_u32, c_u32, c_u32, c_u32, c_u32, c_vp, c_vp, c_vp, c_vp]),
    "ephdc_ctx_create": (c_st, [ctypes.POINTER(Params), c_int, c_vp]),
    "ephdc_ctx_free": (None, [c_vp]),
    "ephdc_ctx_query": (c_st, [c_vp, ctypes.POINTER(CtxInfo)]),
    "ephdc_seed_os": (c_st, [ctypes.POINTER(Seed)]),
    "ephdc_seed_u64": (c_st, [c_u64, ctypes.POINTER(Seed)]),
    "ephdc_chacha20_block": (c_st, [ctypes.POINTER(Seed), c_u32, c_vp, c_vp]),
    "ephdc_keygen": (c_st, [c_vp, ctypes.POINTER(Seed), c_vp]),
    "ephdc_sk_free": (None, [c_vp]),
    "ephdc_sk_export": (c_st, [c_vp, c_vp, c_vp]),
    "ephdc_encrypt_model": (c_st, [c_vp, c_vp, c_vp, ctypes.POINTER(Seed), c_vp]),
    "ephdc_model_free": (None, [c_vp]),
    "ephdc_model_export": (c_st, [c_vp, c_u32, c_u32, c_vp]),
    "ephdc_model_scale": (c_st, [c_vp, c_vp, c_u32, c_vp, c_u32]),
    "ephdc_workspace_create": (c_st, [c_vp, c_u32, c_vp, c_vp]),
    "ephdc_workspace_free": (None, [c_vp]),
    "ephdc_workspace_set_timing": (c_st, [c_vp, c_int]),
    "ephdc_workspace_timing": (c_st, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ephdc_encode_queries": (c_st, [c_vp, c_vp, c_vp, c_u32, c_vp, c_vp]),
    "ephdc_encode_raw": (c_st, [c_vp, c_vp, c_vp, c_u32, c_vp, c_vp]),
    "ephdc_infer_batch": (c_st, [c_vp, c_vp, c_vp, c_vp, c_u32, c_vp, c_u32, c_vp]),
    "ephdc_infer_batch_prefix": (c_st, [c_vp, c_vp, c_vp, c_vp, c_u32, c_vp, c_vp, c_u32, c_vp]),
    "ephdc_encode_plaintexts": (c_st, [c_vp, c_vp, c_vp, c_u32, c_u32, c_u32, c_u32, c_vp, c_vp]),
    "ephdc_classify_host": (c_st, [c_vp, c_vp, c_vp, c_vp, c_vp, c_u32, c_vp, c_u32, c_vp]),
    "ephdc_decrypt_scores": (c_st, [c_vp, c_vp, c_vp, c_u32, c_vp, c_vp]),
    "ephdc_sr_encrypt_queries": (c_st, [c_vp, c_vp, c_vp, c_vp, c_u32, c_u32, ctypes.POINTER(Seed), c_vp, c_vp]),
    "ephdc_sr_model_plaintexts": (c_st, [c_vp, c_vp, c_vp]),
    "ephdc_sr_evaluate": (c_st, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ephdc_scores_message_bytes": (ctypes.c_size_t, [c_vp, c_u32]),
    "ephdc_pack_scores": (c_st, [c_vp, c_vp, c_u32, c_vp, c_vp]),
    "ephdc_unpack_scores": (c_st, [c_vp, c_vp, c_u32, c_vp]),
    "ephdc_classify_host_packed": (c_st, [c_vp, c_vp, c_vp, c_vp, c_vp, c_u32, c_vp, ctypes.c_size_t, c_vp]),
    "ephdc_decrypt_slots": (c_st, [c_vp, c_vp, c_vp, c_vp]),
    "ephdc_noise_probe": (c_st, [c_vp, c_vp, c_vp, c_u32, c_vp, c_vp, c_vp, c_vp]),
    "ephdc_ntt_plan_create": (c_st, [c_vp, c_u32, c_u32, c_int, c_u32, c_vp]),
    "ephdc_ntt_plan_free": (None, [c_vp]),
    "ephdc_ntt_fwd": (c_st, [c_vp, c_vp, c_u32, c_vp]),
    "ephdc_ntt_inv": (c_st, [c_vp, c_vp, c_u32, c_vp]),
    "ephdc_mac": (c_st, [c_vp, c_vp, c_vp, c_u32, c_vp, c_vp]),
    "ephdc_ntt_fwd32": (c_st, [c_vp, c_vp, c_u32, c_vp]),
    "ephdc_ntt_inv32": (c_st, [c_vp, c_vp, c_u32, c_vp]),
    "ephdc_mac32": (c_st, [c_vp, c_vp, c_vp, c_u32, c_vp, c_vp]),
    "ephdc_ntt_plan_query": (c_st, [c_vp, c_vp]),
}

EXPORTED = tuple(_SIGS)


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libephdc.so not found at {LIB_PATH}: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(fn: str, status: int) -> None:
    if status != 0:
        raise EphdcError(fn, status, lib.ephdc_status_string(status).decode())


def call(name: str, *args) -> None:
    check(name, getattr(lib, name)(*args))


def handle() -> ctypes.c_void_p:
    return ctypes.c_void_p()


def launch_count() -> int:
    return int(lib.ephdc_launch_count())


def loaded_path() -> Optional[str]:
    return LIB_PATH
