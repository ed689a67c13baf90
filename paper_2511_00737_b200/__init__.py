"""paper_2511_00737_b200 -- B200 (sm_100a) hot path of EP-HDC client-side encrypted HDC inference.

Python layer over libephdc.so (include/ephdc.h).  PyTorch supplies device memory
and streams; every step of the path runs in the library's CUDA kernels.  Names
follow the C ABI: Context (ephdc_ctx_*), SecretKey (ephdc_keygen), EncryptedModel
(ephdc_encrypt_model), Workspace (ephdc_workspace_*), encode_queries,
infer_batch, decrypt_scores, NttPlan (ephdc_ntt_*), mac.
"""
from __future__ import annotations

import ctypes
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import EphdcError, call, lib

__all__ = [
    "Context", "SecretKey", "EncryptedModel", "Workspace", "NttPlan", "EphdcError", "make_seed", "chacha20_block",
    "find_ntt_primes", "min_psi", "gaussian_cdt", "query_bits", "train_model", "launch_count",
    "encode_queries", "encode_raw", "infer_batch", "infer_batch_prefix", "encode_plaintexts", "classify_host",
    "scores_message_bytes", "pack_scores", "unpack_scores", "classify_host_packed",
    "sr_encrypt_queries", "sr_model_plaintexts", "sr_evaluate",
    "decrypt_scores", "decrypt_slots", "ntt_fwd", "ntt_inv", "mac", "ntt_fwd32", "ntt_inv32", "mac32",
]


def _np_ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def _dptr(t) -> int:
    """Device pointer of a contiguous CUDA torch tensor."""
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return t.data_ptr()


def _stream(stream=None) -> Optional[int]:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def launch_count() -> int:
    return _capi.launch_count()


# --------------------------------------------------------------------------- host helpers
def find_ntt_primes(log2N: int, bits: Sequence[int], exclude: Sequence[int] = ()) -> list:
    b = np.ascontiguousarray(np.array(bits, dtype=np.uint32))
    ex = np.ascontiguousarray(np.array(list(exclude) or [0], dtype=np.uint64))
    out = np.zeros(len(bits), dtype=np.uint64)
    call("ephdc_find_ntt_primes", log2N, _np_ptr(b), len(bits), _np_ptr(ex), len(exclude), _np_ptr(out))
    return [int(x) for x in out]


def min_psi(p: int, log2N: int) -> int:
    out = ctypes.c_uint64()
    call("ephdc_min_psi", p, log2N, ctypes.addressof(out))
    return int(out.value)


def query_bits(D_live: int, Cbits: int, t: int) -> int:
    """ephdc_query_bits: reading #12."""
    out = ctypes.c_uint32()
    call("ephdc_query_bits", D_live, Cbits, t, ctypes.addressof(out))
    return int(out.value)


def train_model(acc_train: np.ndarray, y_train: np.ndarray, k: int, Cbits: int, Qbits: int) -> Tuple[np.ndarray, int]:
    """ephdc_train_model: bundle + quantise the class HVs, calibrate the query shift.
    acc_train int32 [D_live][n]; returns (class_hv int8 [k][D_live], qshift)."""
    acc = np.ascontiguousarray(acc_train, dtype=np.int32)
    lab = np.ascontiguousarray(y_train, dtype=np.int64)
    D, n = acc.shape
    C = np.zeros((k, D), dtype=np.int8)
    s = ctypes.c_uint32()
    call("ephdc_train_model", D, n, k, Cbits, Qbits, _np_ptr(acc), _np_ptr(lab), _np_ptr(C), ctypes.addressof(s))
    return C, int(s.value)


def gaussian_cdt(sigma: float = 3.2) -> np.ndarray:
    out = np.zeros(20, dtype=np.uint64)
    call("ephdc_gaussian_cdt", sigma, _np_ptr(out))
    return out


# --------------------------------------------------------------------------- handles
class Context:
    """ephdc_ctx: parameters, twiddle tables, device constants."""

    def __init__(self, *, log2N: int, q: Sequence[int], t: int, k: int, D_live: int, D_stored: int, F: int,
                 feat_unsigned: bool, Qbits: int, Cbits: int, qshift: int, sigma_e: float = 3.2,
                 device: int = 0, arith: int = 0, encoder: int = 0):
        self._q = np.ascontiguousarray(np.array(q, dtype=np.uint64))
        self.params = _capi.Params(log2N, len(q), self._q.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), t, k,
                                   D_live, D_stored, F, int(feat_unsigned), Qbits, Cbits, qshift, sigma_e, arith,
                                   encoder)
        self._h = ctypes.c_void_p()
        call("ephdc_ctx_create", ctypes.byref(self.params), device, ctypes.byref(self._h))
        info = _capi.CtxInfo()
        call("ephdc_ctx_query", self._h, ctypes.byref(info))
        self.info = info
        self.N, self.L, self.B, self.k = info.N, info.L, info.B, info.k
        self.t, self.psi_t = int(info.t), int(info.psi_t)
        self.q = [int(info.q[j]) for j in range(self.L)]
        self.psi = [int(info.psi[j]) for j in range(self.L)]
        self.delta = [int(info.delta[j]) for j in range(self.L)]
        self.D_live, self.D_stored, self.F = D_live, D_stored, F
        self.feat_unsigned = bool(feat_unsigned)
        self.Qbits, self.Cbits, self.qshift = Qbits, Cbits, qshift
        self.device = device
        self.arith = "f64" if info.arith == _capi.ARITH_F64 else "int"

    @property
    def handle(self):
        return self._h

    def n_batches(self, nq: int) -> int:
        return (nq + self.B - 1) // self.B

    def ct_shape(self, nq: int) -> Tuple[int, int, int, int]:
        return (self.n_batches(nq), 2, self.L, self.N)

    def close(self):
        if self._h:
            lib.ephdc_ctx_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_seed(seed=None):
    """ephdc_seed for the random streams (reading #7).  None: NULL, the library draws a
    fresh 256-bit key from the OS (the default; streams nobody can reproduce); int:
    ephdc_seed_u64 -- DETERMINISTIC and guessable, for parity tests and benchmarks only;
    bytes (32): that key."""
    if seed is None:
        return None
    s = _capi.Seed()
    if isinstance(seed, (bytes, bytearray)):
        if len(seed) != 32:
            raise ValueError("a key seed is 32 bytes")
        ctypes.memmove(s.key, bytes(seed), 32)
    else:
        call("ephdc_seed_u64", int(seed), ctypes.byref(s))
    return ctypes.byref(s)


def chacha20_block(key: bytes, counter: int, nonce) -> np.ndarray:
    """ephdc_chacha20_block: the generator's block function (RFC 8439 sec. 2.3.1), host side."""
    s = _capi.Seed()
    ctypes.memmove(s.key, bytes(key), 32)
    n = np.ascontiguousarray(nonce, dtype=np.uint32)
    out = np.zeros(16, dtype=np.uint32)
    call("ephdc_chacha20_block", ctypes.byref(s), counter, _np_ptr(n), _np_ptr(out))
    return out


class SecretKey:
    def __init__(self, ctx: Context, seed=None):
        """seed: see make_seed (None = OS entropy)."""
        self.ctx = ctx
        self._h = ctypes.c_void_p()
        call("ephdc_keygen", ctx.handle, make_seed(seed), ctypes.byref(self._h))

    @property
    def handle(self):
        return self._h

    def export(self) -> Tuple[np.ndarray, np.ndarray]:
        s = np.zeros(self.ctx.N, dtype=np.int8)
        sh = np.zeros((self.ctx.L, self.ctx.N), dtype=np.uint64)
        call("ephdc_sk_export", self._h, _np_ptr(s), _np_ptr(sh))
        return s, sh

    def __del__(self):
        try:
            if self._h:
                lib.ephdc_sk_free(self._h)
        except Exception:
            pass


class EncryptedModel:
    """ephdc_model: D_live NTT-form ciphertexts resident on the device."""

    def __init__(self, ctx: Context, sk: SecretKey, class_hv: np.ndarray, seed=None):
        C = np.ascontiguousarray(class_hv, dtype=np.int8)
        if C.shape != (ctx.k, ctx.D_live):
            raise ValueError(f"class_hv must be [k, D_live] = {(ctx.k, ctx.D_live)}")
        self.ctx = ctx
        self._h = ctypes.c_void_p()
        call("ephdc_encrypt_model", ctx.handle, sk.handle, _np_ptr(C), make_seed(seed), ctypes.byref(self._h))

    @property
    def handle(self):
        return self._h

    def export(self, d0: int, nd: int) -> np.ndarray:
        out = np.zeros((nd, self.ctx.L, 2, self.ctx.N), dtype=np.uint64)
        call("ephdc_model_export", self._h, d0, nd, _np_ptr(out))
        return out

    def scale(self, g: int, scales: Sequence[int]) -> "EncryptedModel":
        """ephdc_model_scale: fold the accumulator-scaling schedule (one scale per group of
        g dims) into the model, in place."""
        s = np.ascontiguousarray(np.array([int(x) for x in scales] or [1], dtype=np.uint64))
        call("ephdc_model_scale", self.ctx.handle, self._h, g, _np_ptr(s), len(scales))
        return self

    def __del__(self):
        try:
            if self._h:
                lib.ephdc_model_free(self._h)
        except Exception:
            pass


class Workspace:
    """ephdc_workspace.  plan: TEST/PROFILING launch-plan overrides {"flags", "bg", "G",
    "m_batches"} (ephdc_plan; None = the tuned plan, results bit-identical)."""

    def __init__(self, ctx: Context, max_nq: int, plan: Optional[Dict[str, int]] = None):
        self.ctx = ctx
        self.max_nq = max_nq
        pl = dict(plan or {})
        unknown = set(pl) - {"flags", "bg", "G", "m_batches"}
        if unknown:
            raise ValueError(f"unknown plan overrides {sorted(unknown)}")
        self._plan = _capi.Plan(pl.get("flags", 0), pl.get("bg", 0), pl.get("G", 0), pl.get("m_batches", 0))
        self._h = ctypes.c_void_p()
        call("ephdc_workspace_create", ctx.handle, max_nq, ctypes.byref(self._plan), ctypes.byref(self._h))

    @property
    def handle(self):
        return self._h

    def set_timing(self, enable: bool) -> None:
        call("ephdc_workspace_set_timing", self._h, int(enable))

    def timing(self) -> Dict[str, Tuple[float, int]]:
        n = ctypes.c_uint32(8)
        names = (ctypes.c_char_p * 8)()
        ms = np.zeros(8, dtype=np.float64)
        cnt = np.zeros(8, dtype=np.uint64)
        call("ephdc_workspace_timing", self._h, ctypes.addressof(names), _np_ptr(ms), _np_ptr(cnt), ctypes.byref(n))
        return {names[i].decode(): (float(ms[i]), int(cnt[i])) for i in range(n.value)}

    def __del__(self):
        try:
            if self._h:
                lib.ephdc_workspace_free(self._h)
        except Exception:
            pass


# --------------------------------------------------------------------------- client hot path
def encode_queries(ctx: Context, X, P, H=None, stream=None):
    """X: cuda [nq, F] int8/uint8, P: cuda [D_stored, F] int8 -> H cuda [D_live, nq] int8."""
    import torch
    nq = X.shape[0]
    if H is None:
        H = torch.empty((ctx.D_live, nq), dtype=torch.int8, device=X.device)
    call("ephdc_encode_queries", ctx.handle, _dptr(X), _dptr(P), nq, _dptr(H), _stream(stream))
    return H


def encode_raw(ctx: Context, X, P, out=None, stream=None):
    """Unquantised int32 projection acc[d][n] (server-side training; same kernel, RAW epilogue)."""
    import torch
    n = X.shape[0]
    if out is None:
        out = torch.empty((ctx.D_live, n), dtype=torch.int32, device=X.device)
    call("ephdc_encode_raw", ctx.handle, _dptr(X), _dptr(P), n, _dptr(out), _stream(stream))
    return out


def infer_batch(ctx: Context, model: EncryptedModel, ws: Workspace, H, nq: Optional[int] = None, out=None,
                stream=None):
    """H: cuda [D_live, nq] int8 -> scores ciphertexts cuda [nb, 2, L, N] uint64 (as int64 storage)."""
    import torch
    nq = H.shape[1] if nq is None else nq
    if out is None:
        out = torch.empty(ctx.ct_shape(nq), dtype=torch.int64, device=H.device)
    call("ephdc_infer_batch", ctx.handle, model.handle, ws.handle, _dptr(H), nq, _dptr(out), out.shape[0],
         _stream(stream))
    return out


def infer_batch_prefix(ctx: Context, model: EncryptedModel, ws: Workspace, H, nq: int, dims, out=None, stream=None):
    """ephdc_infer_batch_prefix: batch b sums its first dims[b] dims (findDmax's evaluation)."""
    import torch
    nb = ctx.n_batches(nq)
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.uint32))
    assert d.size == nb
    if out is None:
        out = torch.empty(ctx.ct_shape(nq), dtype=torch.int64, device=H.device)
    call("ephdc_infer_batch_prefix", ctx.handle, model.handle, ws.handle, _dptr(H), nq, _np_ptr(d), _dptr(out),
         out.shape[0], _stream(stream))
    return out


def encode_plaintexts(ctx: Context, ws: Workspace, H, b: int, d0: int, nd: int, out=None, stream=None):
    import torch
    nq = H.shape[1]
    if out is None:
        out = torch.empty((nd, ctx.L, ctx.N), dtype=torch.int64, device=H.device)
    call("ephdc_encode_plaintexts", ctx.handle, ws.handle, _dptr(H), nq, b, d0, nd, _dptr(out), _stream(stream))
    return out


def classify_host(ctx: Context, model: EncryptedModel, ws: Workspace, X_host, P, out_host=None, stream=None):
    """End-to-end call with host buffers (X_host: pinned CPU tensor [nq, F]; returns CPU [nb,2,L,N])."""
    import torch
    nq = X_host.shape[0]
    if out_host is None:
        out_host = torch.empty(ctx.ct_shape(nq), dtype=torch.int64, pin_memory=True)
    call("ephdc_classify_host", ctx.handle, model.handle, ws.handle, X_host.data_ptr(), _dptr(P), nq,
         out_host.data_ptr(), out_host.shape[0], _stream(stream))
    return out_host


# --------------------------------------------------------------------------- HE-HDC-SR baseline
def sr_encrypt_queries(ctx: Context, sk: SecretKey, ws: Workspace, H, nq: int, b: int, seed=None, out=None,
                       stream=None):
    """Client of HE-HDC-SR: batch b of H cuda [D_live, nq] -> cuda [D_live, L, 2, N] ciphertexts."""
    import torch
    if out is None:
        out = torch.empty((ctx.D_live, ctx.L, 2, ctx.N), dtype=torch.int64, device=H.device)
    call("ephdc_sr_encrypt_queries", ctx.handle, sk.handle, ws.handle, _dptr(H), nq, b, make_seed(seed), _dptr(out),
         _stream(stream))
    return out


def sr_model_plaintexts(ctx: Context, class_hv: np.ndarray, out=None):
    """Server of HE-HDC-SR, once: plaintext class tiles in NTT form, cuda [D_live, L, N]."""
    import torch
    C = np.ascontiguousarray(class_hv, dtype=np.int8)
    if out is None:
        out = torch.empty((ctx.D_live, ctx.L, ctx.N), dtype=torch.int64, device=torch.device("cuda", ctx.device))
    call("ephdc_sr_model_plaintexts", ctx.handle, _np_ptr(C), _dptr(out))
    return out


def sr_evaluate(ctx: Context, pt, qct, out=None, stream=None):
    """Server of HE-HDC-SR: sum_d qct[d] * pt[d] -> cuda [2, L, N] scores ciphertext."""
    import torch
    if out is None:
        out = torch.empty((2, ctx.L, ctx.N), dtype=torch.int64, device=qct.device)
    call("ephdc_sr_evaluate", ctx.handle, _dptr(pt), _dptr(qct), _dptr(out), _stream(stream))
    return out


# --------------------------------------------------------------------------- scores message
def scores_message_bytes(ctx: Context, nb: int) -> int:
    return int(lib.ephdc_scores_message_bytes(ctx.handle, nb))


def pack_scores(ctx: Context, cts, msg=None, stream=None):
    """cts: cuda [nb, 2, L, N] -> cuda uint8 message (bit-packed residues)."""
    import torch
    nb = cts.shape[0]
    if msg is None:
        msg = torch.empty(scores_message_bytes(ctx, nb), dtype=torch.uint8, device=cts.device)
    call("ephdc_pack_scores", ctx.handle, _dptr(cts), nb, _dptr(msg), _stream(stream))
    return msg


def unpack_scores(ctx: Context, msg: np.ndarray, nb: int) -> np.ndarray:
    m = np.ascontiguousarray(msg, dtype=np.uint8)
    out = np.zeros((nb, 2, ctx.L, ctx.N), dtype=np.uint64)
    call("ephdc_unpack_scores", ctx.handle, _np_ptr(m), nb, _np_ptr(out))
    return out


def classify_host_packed(ctx: Context, model: EncryptedModel, ws: Workspace, X_host, P, msg_host=None, stream=None):
    """End-to-end client call returning the message sent to the server (pinned CPU uint8)."""
    import torch
    nq = X_host.shape[0]
    if msg_host is None:
        msg_host = torch.empty(scores_message_bytes(ctx, ctx.n_batches(nq)), dtype=torch.uint8, pin_memory=True)
    call("ephdc_classify_host_packed", ctx.handle, model.handle, ws.handle, X_host.data_ptr(), _dptr(P), nq,
         msg_host.data_ptr(), msg_host.numel(), _stream(stream))
    return msg_host


# --------------------------------------------------------------------------- server decide (host)
def decrypt_scores(ctx: Context, sk: SecretKey, cts: np.ndarray, nq: int) -> Tuple[np.ndarray, np.ndarray]:
    c = np.ascontiguousarray(cts, dtype=np.uint64)
    scores = np.zeros((nq, ctx.k), dtype=np.int64)
    labels = np.zeros(nq, dtype=np.uint32)
    call("ephdc_decrypt_scores", ctx.handle, sk.handle, _np_ptr(c), nq, _np_ptr(scores), _np_ptr(labels))
    return scores, labels


def decrypt_slots(ctx: Context, sk: SecretKey, ct: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(ct, dtype=np.uint64)
    out = np.zeros(ctx.N, dtype=np.uint64)
    call("ephdc_decrypt_slots", ctx.handle, sk.handle, _np_ptr(c), _np_ptr(out))
    return out


def noise_probe(ctx: Context, sk: SecretKey, cts, stream=None) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """ephdc_noise_probe: per device scores ciphertext of cts [nct][2][L][N] (torch int64
    on the GPU) the exact bit length of the decryption noise, the rounding-ambiguity flag
    and log2 of the noise (findDmax)."""
    nct = int(cts.shape[0]) if cts.dim() == 4 else 1
    bits = np.zeros(nct, dtype=np.uint32)
    flags = np.zeros(nct, dtype=np.uint32)
    lg = np.zeros(nct, dtype=np.float64)
    call("ephdc_noise_probe", ctx.handle, sk.handle, _dptr(cts), nct, _np_ptr(bits), _np_ptr(flags), _np_ptr(lg),
         _stream(stream))
    return bits, flags, lg


# --------------------------------------------------------------------------- standalone (c5)
class NttPlan:
    """ephdc_ntt_plan.  force_int: the integer-pipe kernels everywhere (EPHDC_NTT_FORCE_INT);
    alt_teams: the other warp layout of the c5 kernels at N = 2^13 (EPHDC_NTT_ALT_TEAMS); u32_generic:
    the general u32 kernels instead of the TMA-fed ones of ntt32_c5.cu (EPHDC_NTT_U32_GENERIC).  All are
    tests/profiling switches with bit-identical results."""

    def __init__(self, q: Sequence[int], log2N: int, device: int = 0, force_int: bool = False,
                 alt_teams: bool = False, u32_generic: bool = False):
        self.q = [int(x) for x in q]
        self.L, self.log2N, self.N = len(q), log2N, 1 << log2N
        qa = np.ascontiguousarray(np.array(self.q, dtype=np.uint64))
        self._h = ctypes.c_void_p()
        call("ephdc_ntt_plan_create", _np_ptr(qa), self.L, log2N, device,
             (1 if force_int else 0) | (2 if alt_teams else 0) | (4 if u32_generic else 0), ctypes.byref(self._h))
        info = (ctypes.c_uint32 * 4)()
        call("ephdc_ntt_plan_query", self._h, ctypes.addressof(info))
        names = {0: "int", 1: "f64", 2: "c5_f64", 3: "c5_u32"}
        self.fwd_kernel, self.inv_kernel = names[info[0]], names[info[1]]
        self.u32_words = bool(info[2])
        self.u32_kernel = ("int_u32" if info[3] == 0 else names[info[3]]) if self.u32_words else None

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                lib.ephdc_ntt_plan_free(self._h)
        except Exception:
            pass


def ntt_fwd(plan: NttPlan, polys, stream=None):
    call("ephdc_ntt_fwd", plan.handle, _dptr(polys), polys.numel() // (plan.L * plan.N), _stream(stream))
    return polys


def ntt_inv(plan: NttPlan, polys, stream=None):
    call("ephdc_ntt_inv", plan.handle, _dptr(polys), polys.numel() // (plan.L * plan.N), _stream(stream))
    return polys


def ntt_fwd32(plan: NttPlan, polys, stream=None):
    """u32 words (torch.int32 storage of residues < 2^30)."""
    call("ephdc_ntt_fwd32", plan.handle, _dptr(polys), polys.numel() // (plan.L * plan.N), _stream(stream))
    return polys


def ntt_inv32(plan: NttPlan, polys, stream=None):
    call("ephdc_ntt_inv32", plan.handle, _dptr(polys), polys.numel() // (plan.L * plan.N), _stream(stream))
    return polys


def mac32(plan: NttPlan, ct, pt, out=None, stream=None):
    import torch
    D = pt.shape[0]
    if out is None:
        out = torch.empty((plan.L, 2, plan.N), dtype=torch.int32, device=pt.device)
    call("ephdc_mac32", plan.handle, _dptr(ct), _dptr(pt), D, _dptr(out), _stream(stream))
    return out


def mac(plan: NttPlan, ct, pt, out=None, stream=None):
    import torch
    D = pt.shape[0]
    if out is None:
        out = torch.empty((plan.L, 2, plan.N), dtype=torch.int64, device=pt.device)
    call("ephdc_mac", plan.handle, _dptr(ct), _dptr(pt), D, _dptr(out), _stream(stream))
    return out
