"""FP8 E4M3 decoding and attention over an FP8 KV cache -- TEST INFRASTRUCTURE ONLY.

The FP8 cache row of SURVEY.md §8(f) (f4) goes beyond the paper (fp16 only), so its
oracle is the same plain attention (oracle.attention) over the DECODED
cache: K = k_scale[g] * E4M3(K8), V = v_scale[g] * E4M3(V8) for KV head g.

E4M3 (the OCP 8-bit floating point "E4M3" format, the fn variant without infinities), written out
from its definition: bit 7 sign, bits 6-3 exponent e (bias 7), bits 2-0 mantissa m;
  e = 0        : (-1)^s * (m / 8) * 2^-6          (subnormal; m = 0 is +-0)
  e = 1..15    : (-1)^s * (1 + m / 8) * 2^(e - 7)  except e = 15, m = 7: NaN (max finite 448).
"""
from __future__ import annotations

import math

import numpy as np


def e4m3_value(byte: int) -> float:
    """Value of one E4M3 byte (the definition above, one case per line)."""
    s = -1.0 if byte & 0x80 else 1.0
    e = (byte >> 3) & 0xF
    m = byte & 0x7
    if e == 15 and m == 7:
        return math.nan
    if e == 0:
        return s * (m / 8.0) * 2.0 ** -6
    return s * (1.0 + m / 8.0) * 2.0 ** (e - 7)


E4M3_TABLE = np.array([e4m3_value(b) for b in range(256)], dtype=np.float64)


def decode_e4m3(bytes_u8) -> np.ndarray:
    """float64 values of an array of E4M3 bytes (uint8, any shape)."""
    a = np.asarray(bytes_u8.cpu() if hasattr(bytes_u8, "cpu") else bytes_u8, dtype=np.uint8)
    return E4M3_TABLE[a]


def decode_cache(k8, scale) -> np.ndarray:
    """Decoded cache [B, N, H_kv, d] = scale[g] * E4M3(k8) in float64.  The tests use power-of-two
    scales, so the values are also exact in float32 (the oracle's input precision)."""
    sc = np.asarray(scale.cpu() if hasattr(scale, "cpu") else scale, dtype=np.float64)
    return decode_e4m3(k8) * sc[None, None, :, None]


def attention_fp8kv(q, k8, v8, k_scale, v_scale, k_tree, v_tree, mask, **kw):
    """oracle.attention over the decoded E4M3 cache (k_scale / v_scale powers of two, checked)."""
    from .attention import attention
    for sc in (k_scale, v_scale):
        a = np.asarray(sc.cpu() if hasattr(sc, "cpu") else sc, dtype=np.float64)
        m, _ = np.frexp(a)
        if not np.all(m == 0.5):
            raise ValueError("the FP8 oracle takes power-of-two scales (exact decoded values in float32)")
    kc = decode_cache(k8, k_scale).astype(np.float32)
    vc = decode_cache(v8, v_scale).astype(np.float32)
    return attention(q, kc, vc, k_tree, v_tree, mask, **kw)
