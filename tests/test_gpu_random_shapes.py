"""Seeded random sweep of shapes vs the fp64 oracle: batch, tree size, GQA group (including
G that does not divide 128, so Q is staged by loads), head dim, prefix length (ragged tails,
lengths shorter than one tile), per-batch cache_seqlens (including 0), trees of every generator
shape and the three value distributions -- hta_forward and its two partials."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload

from gpu_util import compare, oracle_masks, to_dev

pytestmark = pytest.mark.gpu

TREES = ["beam", "random", "chain", "star", "roots", "random_forest", "heap_binary"]


def _case(i):
    r = np.random.default_rng(1000 + i)
    d = int(r.choice([64, 128]))
    Hkv = int(r.choice([1, 2, 4, 8]))
    G = int(r.choice([1, 2, 3, 4, 5, 6, 8]))
    T = int(r.choice([1, 3, 8, 16, 31, 64, 100]))
    B = int(r.integers(1, 4))
    N = int(r.choice([5, 150, 193, 700, 1500, 3100]))
    dist = str(r.choice(["V0", "V1", "V2"]))
    tree = str(r.choice(TREES))
    return B, T, Hkv * G, Hkv, d, N, dist, tree


@pytest.mark.parametrize("i", range(24))
def test_random_shape(cuda_device, i):
    B, T, H, Hkv, d, N, dist, tree = _case(i)
    if tree == "heap_binary" and T > 64:
        tree = "random"
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist=dist, seed=50 + i, tree=tree)
    rng = np.random.default_rng(i)
    sl = torch.from_numpy(rng.integers(0, N + 1, size=B).astype(np.int32))
    sl[0] = N  # at least one full-length batch entry
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    sl_d = sl.to(cuda_device)
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                           cache_seqlens=sl_d)
    oc, lc = hta.hta_prefix_attn(x["q"], x["kc"], x["vc"], cache_seqlens=sl_d)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=sl)
    oc_ref, lc_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=sl, part="cache")
    desc = f"B{B} T{T} H{H}/{Hkv} d{d} N{N} {dist} {tree} sl={sl.tolist()}"
    compare(o, l, o_ref, l_ref, "bf16", "forward " + desc)
    compare(oc, lc, oc_ref, lc_ref, "bf16", "prefix " + desc)
