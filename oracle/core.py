"""ctypes binding of oracle_core.c (gcc-built) -- TEST INFRASTRUCTURE ONLY."""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle_core.c")
_LIB = os.path.join(_HERE, "liboracle.so")

u64 = ctypes.c_uint64
u32 = ctypes.c_uint32
P = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle_core.c with gcc (plain -O2, OpenMP over independent dims)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class OrBfv(ctypes.Structure):
    _fields_ = [
        ("logN", ctypes.c_int), ("L", u32), ("q", P), ("psi", P), ("t", u64), ("psi_t", u64),
        ("k", u32), ("D_live", u32), ("delta", P), ("s_hat", P), ("enc_seed", u64),
        ("cdt", P), ("ncdt", ctypes.c_int),
    ]


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        sig = {
            "or_mulmod": (u64, [u64, u64, u64]),
            "or_powmod": (u64, [u64, u64, u64]),
            "or_brev": (u32, [u32, ctypes.c_int]),
            "or_pow_brev_table": (None, [u64, u64, ctypes.c_int, P]),
            "or_ntt_fwd": (None, [P, ctypes.c_int, u64, P]),
            "or_ntt_inv": (None, [P, ctypes.c_int, u64, P]),
            "or_ntt_fwd_many": (None, [P, u64, ctypes.c_int, u64, u64]),
            "or_ntt_inv_many": (None, [P, u64, ctypes.c_int, u64, u64]),
            "or_eval": (u64, [P, u32, u64, u64]),
            "or_negacyclic_mul": (None, [P, P, P, u32, u64]),
            "or_chacha20_block": (None, [P, u32, P, P]),
            "or_word64": (u64, [u64, u32, u64, u32, u32]),
            "or_sample_ternary": (None, [u64, u32, P]),
            "or_uniform_mod": (u64, [u64, u64, u32, u32, u32, u64]),
            "or_gauss": (ctypes.c_longlong, [u64, u64, u32, P, ctypes.c_int]),
            "or_sample_uniform_poly": (None, [u64, u64, u32, u32, u64, u32, P]),
            "or_sample_gauss_poly": (None, [u64, u64, u32, P, ctypes.c_int, P]),
            "or_encrypt_dims": (None, [ctypes.POINTER(OrBfv), P, u32, u32, P]),
            "or_plaintext_ntts": (None, [ctypes.POINTER(OrBfv), P, u32, u32, u32, u32, P]),
            "or_infer_batch": (None, [ctypes.POINTER(OrBfv), P, u32, u32, P, P, P, P]),
            "or_infer_batch_range": (None, [ctypes.POINTER(OrBfv), P, u32, u32, u32, u32, P, P, P, P]),
            "or_encrypt_queries": (None, [ctypes.POINTER(OrBfv), P, u32, u32, u32, u32, P]),
            "or_server_eval": (None, [ctypes.POINTER(OrBfv), P, P, P]),
            "or_decrypt_phase": (None, [ctypes.POINTER(OrBfv), P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def u64arr(x: Sequence[int]) -> np.ndarray:
    return np.ascontiguousarray(np.array([int(v) for v in x], dtype=np.uint64))


# -- thin numpy wrappers ---------------------------------------------------------

def pow_brev_table(x: int, q: int, logN: int) -> np.ndarray:
    out = np.empty(1 << logN, dtype=np.uint64)
    lib().or_pow_brev_table(x, q, logN, ptr(out))
    return out


def ntt_fwd(polys: np.ndarray, logN: int, q: int, psi: int) -> np.ndarray:
    a = np.ascontiguousarray(polys, dtype=np.uint64).copy()
    n = a.size >> logN
    lib().or_ntt_fwd_many(ptr(a), n, logN, q, psi)
    return a


def ntt_inv(polys: np.ndarray, logN: int, q: int, psi: int) -> np.ndarray:
    a = np.ascontiguousarray(polys, dtype=np.uint64).copy()
    n = a.size >> logN
    lib().or_ntt_inv_many(ptr(a), n, logN, q, psi)
    return a


def evaluate(poly: np.ndarray, q: int, x: int) -> int:
    a = np.ascontiguousarray(poly, dtype=np.uint64)
    return int(lib().or_eval(ptr(a), a.size, q, x))


def negacyclic_mul(a: np.ndarray, b: np.ndarray, q: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.empty_like(a)
    lib().or_negacyclic_mul(ptr(a), ptr(b), ptr(c), a.size, q)
    return c
