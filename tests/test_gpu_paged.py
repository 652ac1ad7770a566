"""hta_forward_paged (the block-table KV layout of flash_attn_with_kvcache,
PAPER.md:108, for batched serving) vs the fp64 oracle on the gathered cache, and bit-identical to
hta_forward on the contiguous cache (same tiles, same order); pages shuffled across batches,
ragged lengths, page sizes 16..256, both row-group layouts (pairs and single CTAs)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload

from gpu_util import compare, oracle_masks, to_dev

pytestmark = pytest.mark.gpu


def paged(w, page_size, seed, dev):
    """Scatter each batch's cache rows into shuffled pages of one pool; returns (k_pool, v_pool,
    block_table [B, max_pages])."""
    B, N, Hkv, d = w.k_cache.shape
    max_pages = (N + page_size - 1) // page_size
    num_pages = B * max_pages + 3
    rng = np.random.default_rng(seed)
    perm = rng.permutation(num_pages)[:B * max_pages].reshape(B, max_pages)
    kp = torch.zeros(num_pages, page_size, Hkv, d, dtype=w.k_cache.dtype)
    vp = torch.full((num_pages, page_size, Hkv, d), float("nan"), dtype=w.v_cache.dtype)  # unused pages: NaN
    for b in range(B):
        for pg in range(max_pages):
            lo, hi = pg * page_size, min(N, (pg + 1) * page_size)
            kp[perm[b, pg], :hi - lo] = w.k_cache[b, lo:hi]
            vp[perm[b, pg], :hi - lo] = w.v_cache[b, lo:hi]
    return kp.to(dev), vp.to(dev), torch.from_numpy(perm.astype(np.int32)).to(dev)


@pytest.mark.parametrize("case", [
    (2, 64, 32, 8, 128, 3000, 16),    # pairs (M = 256), vLLM-sized pages
    (3, 13, 8, 2, 128, 1000, 64),     # single CTAs, ragged tail
    (1, 40, 10, 2, 128, 2300, 256),   # pages larger than a KV tile
    (2, 17, 4, 1, 64, 900, 32),       # d = 64
])
def test_paged_forward(cuda_device, case):
    B, T, H, Hkv, d, N, page = case
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist="V1", seed=13, tree="beam")
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    m_dev = torch.from_numpy(mask).to(cuda_device)
    kp, vp, bt = paged(w, page, seed=5, dev=cuda_device)
    o_p, l_p = hta.hta_forward_paged(x["q"], kp, vp, bt, x["kt"], x["vt"], m_dev, cache_seqlens=x["sl"])
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    compare(o_p, l_p, o_ref, l_ref, "bf16", f"paged {case}")
    # the same cache gathered back from the pool into a contiguous [B, max_pages * page] cache:
    # the same split plan, tiles and order -> bit-identical to the contiguous forward
    idx = bt.long()
    kc = kp[idx].reshape(B, -1, Hkv, d)
    vc = vp[idx].reshape(B, -1, Hkv, d)
    o_c, l_c = hta.hta_forward(x["q"], kc, vc, x["kt"], x["vt"], m_dev, cache_seqlens=x["sl"])
    torch.cuda.synchronize()
    assert torch.equal(o_p, o_c) and torch.equal(l_p, l_c)
