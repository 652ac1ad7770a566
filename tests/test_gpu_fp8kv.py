"""FP8 (E4M3) KV cache: hta_forward_fp8kv / hta_prefix_attn_fp8kv vs the fp64
oracle over the DECODED cache (oracle.attention_fp8kv), at the bf16 tolerances (DESIGN.md "FP8 KV
cache": the E4M3 -> f16 and bf16 q -> f16 conversions are exact, P is rounded to f16, so the
error budget is the bf16 path's).  Shapes cover CTA pairs (M = 256), single CTAs (MHA M = 64,
G = 5), d = 64, ragged tails with NaN bytes past cache_seqlens, and a logit jump past the f16
range of the speculative exponentials."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import fp8_cache, make_workload
from workloads.generators import named_generator

from gpu_util import compare, oracle_masks

pytestmark = pytest.mark.gpu

CASES = [
    # B, T, H, Hkv, d, N, dist, tree
    (1, 64, 32, 8, 128, 3000, "V1", "beam"),     # pair (M = 256)
    (1, 64, 8, 8, 128, 2500, "V1", "beam"),      # MHA, M = 64 (LongChat-like rows)
    (2, 64, 10, 2, 128, 1500, "V2", "beam"),     # G = 5: single CTAs, three row groups
    (2, 17, 4, 1, 64, 1100, "V1", "star"),       # d = 64
    (1, 30, 6, 2, 128, 900, "V0", "random"),     # G = 3 (Q staged by loads anyway)
    (1, 1, 4, 4, 128, 1, "V1", "chain"),         # single key
]


def _fp8(w, dev):
    k8, ks = fp8_cache(w.k_cache)
    v8, vs = fp8_cache(w.v_cache)
    return k8, ks, v8, vs, {"k8": k8.to(dev), "v8": v8.to(dev), "ks": ks.to(dev), "vs": vs.to(dev)}


@pytest.mark.parametrize("case", CASES, ids=lambda c: "B{}T{}H{}kv{}d{}N{}-{}-{}".format(*c))
def test_fp8kv_forward_and_prefix_vs_oracle(cuda_device, case):
    B, T, H, Hkv, d, N, dist, tree = case
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist=dist, seed=23, tree=tree)
    mask = oracle_masks(w)
    k8, ks, v8, vs, x = _fp8(w, cuda_device)
    o_ref, l_ref = oracle.attention_fp8kv(w.q, k8, v8, ks, vs, w.k_tree, w.v_tree, mask)
    oc_ref, lc_ref = oracle.attention_fp8kv(w.q, k8, v8, ks, vs, w.k_tree, w.v_tree, mask, part="cache")
    q = w.q.to(cuda_device)
    o, l = hta.hta_forward_fp8kv(q, x["k8"], x["v8"], x["ks"], x["vs"], w.k_tree.to(cuda_device),
                                 w.v_tree.to(cuda_device), torch.from_numpy(mask).to(cuda_device))
    oc, lc = hta.hta_prefix_attn_fp8kv(q, x["k8"], x["v8"], x["ks"], x["vs"])
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", "fp8 forward")
    compare(oc, lc, oc_ref, lc_ref, "bf16", "fp8 prefix")


def test_fp8kv_nan_bytes_past_seqlens(cuda_device):
    """E4M3 NaN bytes (0x7F / 0xFF) in every row past cache_seqlens must not reach the result
    (reading Z13): they are masked in S and zeroed while widening V."""
    sl = torch.tensor([1000, 0, 129, 1], dtype=torch.int32)
    w = make_workload(4, 9, 8, 2, 128, 1024, "bf16", dist="V1", seed=5, tree="random", seqlens=sl)
    mask = oracle_masks(w)
    k8, ks, v8, vs, _ = _fp8(w, cuda_device)
    for b in range(4):
        k8[b, int(sl[b]):] = 0x7F
        v8[b, int(sl[b]):] = 0xFF
    o_ref, l_ref = oracle.attention_fp8kv(w.q, k8, v8, ks, vs, w.k_tree, w.v_tree, mask, seqlens=sl)
    for splits in (0, 3):
        o, l = hta.hta_forward_fp8kv(w.q.to(cuda_device), k8.to(cuda_device), v8.to(cuda_device), ks.to(cuda_device),
                                     vs.to(cuda_device), w.k_tree.to(cuda_device), w.v_tree.to(cuda_device),
                                     torch.from_numpy(mask).to(cuda_device), cache_seqlens=sl.to(cuda_device),
                                     num_splits=splits)
        torch.cuda.synchronize()
        compare(o, l, o_ref, l_ref, "bf16", f"fp8 NaN tail splits={splits}")


@pytest.mark.parametrize("key", [3, 130, 300])
def test_fp8kv_logit_jump_past_f16_range(cuda_device, key):
    """A key whose logit exceeds the running max of the earlier tiles by far more than 2^15 in P:
    the f16 speculative exponentials overflow and the tile is redone with its true max."""
    B, T, H, Hkv, d, N = 1, 4, 4, 1, 128, 448
    gen = named_generator(31, f"fp8jump:{key}")
    u = torch.randn(d, generator=gen)
    u = u / u.norm()
    q = (40.0 * u + 0.5 * torch.randn(B, T, H, d, generator=gen)).to(torch.bfloat16)
    kc = torch.randn(B, N, Hkv, d, generator=gen)
    kc[:, key, :, :] = 42.5 * u + 0.1 * kc[:, key, :, :]
    vc = torch.randn(B, N, Hkv, d, generator=gen)
    k8, ks = fp8_cache(kc)
    v8, vs = fp8_cache(vc)
    kt = torch.zeros(B, T, Hkv, d, dtype=torch.bfloat16)
    mask = np.ones((B, T, T), np.uint8)
    oc_ref, lc_ref = oracle.attention_fp8kv(q, k8, v8, ks, vs, kt, kt, mask, part="cache")
    dev = cuda_device
    oc, lc = hta.hta_prefix_attn_fp8kv(q.to(dev), k8.to(dev), v8.to(dev), ks.to(dev), vs.to(dev))
    torch.cuda.synchronize()
    compare(oc, lc, oc_ref, lc_ref, "bf16", "fp8 jump")


@pytest.mark.parametrize("spread", ["rows", "elements"])
def test_fp8kv_q_dynamic_range(cuda_device, spread):
    """Single-CTA units with d = 128 compute S on kind::f8f6f4 with q split into two E4M3 terms at
    one power-of-two scale per CTA.  q rows (or elements within a row) spanning
    ~2^14 in magnitude, and values large enough to need the scale (|q| up to 300), must still meet
    the bf16 tolerances against the oracle over the exact bf16 q."""
    w = make_workload(2, 64, 8, 8, 128, 1500, "bf16", dist="V1", seed=31, tree="beam")
    g = torch.Generator().manual_seed(5)
    if spread == "rows":  # row scales 2^-7 .. 2^7 (per token, all heads)
        f = torch.pow(2.0, torch.randint(-7, 8, (2, 64, 1, 1), generator=g).float())
    else:  # element scales 2^-7 .. 2^7 within every row
        f = torch.pow(2.0, torch.randint(-7, 8, (2, 64, 8, 128), generator=g).float())
    q = (w.q.float() * f * 0.05).to(torch.bfloat16)
    q[0, 0, 0, 0] = 300.0  # one large element: the CTA scale must keep it in E4M3 range
    w.q = q
    mask = oracle_masks(w)
    k8, ks, v8, vs, x = _fp8(w, cuda_device)
    o_ref, l_ref = oracle.attention_fp8kv(w.q, k8, v8, ks, vs, w.k_tree, w.v_tree, mask)
    o, l = hta.hta_forward_fp8kv(w.q.to(cuda_device), x["k8"], x["v8"], x["ks"], x["vs"],
                                 w.k_tree.to(cuda_device), w.v_tree.to(cuda_device),
                                 torch.from_numpy(mask).to(cuda_device))
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", f"fp8 q spread {spread}")


@pytest.mark.parametrize("dist", ["V0", "V1"])
def test_fp8kv_long_context_split_p(cuda_device, dist):
    """Single-CTA units of more than 64 rows run PV on kind::f8f6f4 with P as an E4M3 term plus an
    E5M2 remainder.  A 16k-key context spreads the softmax over many small P
    values (down to E5M2's floor); the bf16 tolerances must still hold against the oracle."""
    w = make_workload(1, 64, 16, 8, 128, 16384, "bf16", dist=dist, seed=37, tree="beam")
    mask = oracle_masks(w)
    k8, ks, v8, vs, x = _fp8(w, cuda_device)
    o_ref, l_ref = oracle.attention_fp8kv(w.q, k8, v8, ks, vs, w.k_tree, w.v_tree, mask)
    o, l = hta.hta_forward_fp8kv(w.q.to(cuda_device), x["k8"], x["v8"], x["ks"], x["vs"],
                                 w.k_tree.to(cuda_device), w.v_tree.to(cuda_device),
                                 torch.from_numpy(mask).to(cuda_device))
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", f"fp8 split-P {dist}")
