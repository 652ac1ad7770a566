"""Pins of the FP8 (E4M3) decoding used by the FP8-cache oracle (oracle/fp8.py), on CPU."""
import math

import numpy as np
import torch

import oracle
from oracle.fp8 import E4M3_TABLE, decode_cache
from workloads import fp8_cache, make_workload


def test_e4m3_closed_forms():
    """Values the format's definition fixes: max finite, min normal, min subnormal, one, sign, NaN."""
    assert oracle.e4m3_value(0x7E) == 448.0
    assert oracle.e4m3_value(0x08) == 2.0 ** -6
    assert oracle.e4m3_value(0x01) == 2.0 ** -9
    assert oracle.e4m3_value(0x07) == 7 * 2.0 ** -9
    assert oracle.e4m3_value(0x38) == 1.0 and oracle.e4m3_value(0xB8) == -1.0
    assert oracle.e4m3_value(0x00) == 0.0 and math.copysign(1.0, oracle.e4m3_value(0x80)) == -1.0
    assert math.isnan(oracle.e4m3_value(0x7F)) and math.isnan(oracle.e4m3_value(0xFF))
    finite = E4M3_TABLE[np.isfinite(E4M3_TABLE)]
    assert len(finite) == 254 and len(np.unique(finite)) == 253  # +-0 coincide


def test_e4m3_table_matches_library_conversion():
    """All 256 bytes decode as torch's float8_e4m3fn (a library routine) does."""
    b = torch.arange(256, dtype=torch.uint8)
    lib = b.view(torch.float8_e4m3fn).to(torch.float64).numpy()
    ours = E4M3_TABLE
    nan = np.isnan(lib)
    assert np.array_equal(nan, np.isnan(ours))
    assert np.array_equal(lib[~nan], ours[~nan])


def test_fp8_cache_generator_roundtrip():
    """The generator's power-of-two scales keep every decoded value within E4M3 rounding of the
    source (relative 2^-4 for normals) and exactly representable in float32."""
    w = make_workload(1, 4, 8, 2, 128, 300, "bf16", dist="V1", seed=2)
    k8, ks = fp8_cache(w.k_cache)
    m, _ = np.frexp(ks.numpy().astype(np.float64))
    assert np.all(m == 0.5)
    dec = decode_cache(k8, ks)
    assert np.array_equal(dec.astype(np.float32).astype(np.float64), dec)
    src = w.k_cache.double().numpy()
    big = np.abs(src) > 0.05
    assert np.all(np.abs(dec[big] - src[big]) <= 2.0 ** -4 * np.abs(src[big]) + 1e-12)
