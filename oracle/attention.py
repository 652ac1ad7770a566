"""fp64 explicit-mask attention and LSE merge -- TEST INFRASTRUCTURE ONLY.

`attention` wraps hta_oracle.c (steps O1-O7, see that file's header).  `merge` is the
aggregation of PAPER.md:203-219 / Appendix C:

    LSE_m = log(exp(LSE_a) + exp(LSE_b))
    O_m   = O_a * exp(LSE_a - LSE_m) + O_b * exp(LSE_b - LSE_m)

written in the max-shifted form (reading Z11: m = max(LSE_a, LSE_b),
LSE_m = m + log(exp(LSE_a - m) + exp(LSE_b - m)), identical in exact arithmetic) and
folded left over any number of parts.  A part whose LSE is -inf
is the empty-part sentinel (O = 0, LSE = -inf, reading Z10) and is the merge identity.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hta_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_library(force: bool = False) -> str:
    """Compile hta_oracle.c with plain gcc -O2 (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off",
                               "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def load_library():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_library())
        lib.oracle_attention.restype = ctypes.c_int
        P = ctypes.c_void_p
        lib.oracle_attention.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long,
            ctypes.c_double, P, P, P, P, P, P, P, ctypes.c_int, ctypes.c_long, ctypes.c_long,
            P, ctypes.c_long, P, P, ctypes.c_int]
        _lib = lib
    return _lib


def _f32(x) -> np.ndarray:
    """Exact float32 copy of a torch tensor / array (bf16 and fp32 values are exact)."""
    if hasattr(x, "detach"):
        import torch
        x = x.detach().to("cpu")
        if x.dtype != torch.float32:
            x = x.to(torch.float32)
        x = x.numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def attention(q, k_cache, v_cache, k_tree, v_tree, mask, seqlens=None, scale: Optional[float] = None,
              part: str = "all", cache_range: Optional[Tuple[int, int]] = None,
              rows: Optional[Sequence[Tuple[int, int, int]]] = None,
              threads: Optional[int] = None):
    """Explicit-mask attention of every (b, t, h) row (or only `rows`).

    q [B,T,H,d]; k_cache/v_cache [B,N,H_kv,d]; k_tree/v_tree [B,T,H_kv,d]; mask uint8
    [B,T,T] (1 = visible); seqlens int [B] or None (= N).  `scale` defaults to
    1/sqrt(d) rounded to float32 (reading Z2: the exact value the kernels see).
    part = "all" | "cache" | "tree" (O7).  cache_range = (lo, hi) restricts the visible
    cache columns (a P-way sequence split).
    Returns (O float64 [B,T,H,d] or [R,d], LSE float64 [B,H,T] or [R]).
    """
    lib = load_library()
    qf, kcf, vcf = _f32(q), _f32(k_cache), _f32(v_cache)
    B, T, H, d = qf.shape
    N, Hkv = kcf.shape[1], kcf.shape[2]
    ktf, vtf = _f32(k_tree), _f32(v_tree)
    if ktf.size == 0:
        ktf = np.zeros((B, max(T, 1), Hkv, d), np.float32)
        vtf = ktf
    m = np.ascontiguousarray(np.asarray(mask.cpu() if hasattr(mask, "cpu") else mask, dtype=np.uint8))
    if m.ndim == 2:
        m = np.ascontiguousarray(np.broadcast_to(m, (B, T, T)))
    if m.size == 0:
        m = np.zeros((B, max(T, 1), max(T, 1)), np.uint8)
    sl = None
    if seqlens is not None:
        sl = np.ascontiguousarray(np.asarray(seqlens.cpu() if hasattr(seqlens, "cpu") else seqlens,
                                             dtype=np.int32))
    if scale is None:
        scale = float(np.float32(1.0 / np.sqrt(d)))
    part_id = {"all": 0, "cache": 1, "tree": 2}[part]
    lo, hi = (0, N) if cache_range is None else cache_range
    if rows is not None:
        ra = np.ascontiguousarray(np.asarray(rows, dtype=np.int32).reshape(-1, 3))
        R = ra.shape[0]
        o = np.zeros((R, d), np.float64)
        lse = np.zeros((R,), np.float64)
    else:
        ra = None
        R = B * T * H
        o = np.zeros((B, T, H, d), np.float64)
        lse_bth = np.zeros((B, T, H), np.float64)
    nthreads = threads or max(1, len(os.sched_getaffinity(0)))
    rc = lib.oracle_attention(B, T, H, Hkv, d, N, float(scale), _ptr(qf), _ptr(kcf), _ptr(vcf), _ptr(sl),
                              _ptr(ktf), _ptr(vtf), _ptr(m), part_id, int(lo), int(hi),
                              _ptr(ra), R, _ptr(o), _ptr(lse if ra is not None else lse_bth), nthreads)
    if rc != 0:
        raise ValueError("oracle_attention: invalid arguments")
    if ra is not None:
        return o, lse
    return o, np.ascontiguousarray(lse_bth.transpose(0, 2, 1))  # -> [B, H, T]


def merge(parts):
    """Fold the LSE aggregation over a list of (O, LSE) parts.

    O arrays are [..., d] and LSE arrays the matching [...] (same leading shape).  Returns
    (O, LSE) in float64.
    """
    o_acc = np.asarray(parts[0][0], np.float64).copy()
    l_acc = np.asarray(parts[0][1], np.float64).copy()
    for o_b, l_b in parts[1:]:
        o_b = np.asarray(o_b, np.float64)
        l_b = np.asarray(l_b, np.float64)
        m = np.maximum(l_acc, l_b)
        empty = np.isneginf(m)
        m_safe = np.where(empty, 0.0, m)
        with np.errstate(invalid="ignore", over="ignore"):
            l_new = m_safe + np.log(np.exp(l_acc - m_safe) + np.exp(l_b - m_safe))
            l_new = np.where(empty, -np.inf, l_new)
            l_ref = np.where(empty, 0.0, l_new)
            w_a = np.where(empty, 0.0, np.exp(l_acc - l_ref))
            w_b = np.where(empty, 0.0, np.exp(l_b - l_ref))
        o_acc = o_acc * w_a[..., None] + o_b * w_b[..., None]
        l_acc = l_new
    return o_acc, l_acc
