"""GPU parity of the fused split combine: the prefix kernel's CTAs of a unit
wait for each other on the unit's arrival counter and merge their rows themselves (tree pass of
CTA-pair units included) instead of a second kernel.

Checked against the oracle AND against the two-kernel path (hta_set_fused_merge(0)) on the
same inputs: both read the same split partials, so they agree to the rounding of the tree pass's
key batching.  Shapes cover CTA pairs and single CTAs, several row groups (G = 5: two waves of
CTAs), T = 128 / 256 (several rows per warp), forced split counts up to a unit of 128 CTAs,
empty splits (short and zero cache_seqlens with NaN garbage past them), the parent-array entry
point and the paged cache; the counter block must be zero again after every call and its error
word never set; CUDA-graph replays must be bit-identical (the counters re-arm themselves).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload, tree_parents

from gpu_util import compare, oracle_masks, to_dev

pytestmark = pytest.mark.gpu


def _ctr_block(ws, shape):
    """The unit counters + error word at the end of the workspace (include/hta.h)."""
    G = shape.H // shape.H_kv
    units = shape.B * shape.H_kv * ((shape.T * G + 127) // 128)
    nbytes = ((2 * units + 1) * 4 + 15) // 16 * 16
    off = (ws.numel() - nbytes) // 16 * 16
    return ws[off:off + (2 * units + 1) * 4].view(torch.int32)


def _both(fn):
    """fn() with the fused merge on (default) and off; returns (fused, two-kernel)."""
    prev = hta.set_fused_merge(True)
    try:
        a = fn()
        torch.cuda.synchronize()
        hta.set_fused_merge(False)
        b = fn()
        torch.cuda.synchronize()
    finally:
        hta.set_fused_merge(prev)
    return a, b


def _close(a, b, what):
    (oa, la), (ob, lb) = a, b
    assert torch.equal(torch.isneginf(la), torch.isneginf(lb)), f"{what}: sentinel rows differ"
    fin = torch.isfinite(la)
    dl = (la[fin] - lb[fin]).abs().max().item() if fin.any() else 0.0
    do = (oa.float() - ob.float()).abs().max().item()
    assert dl <= 1e-4 and do <= 8e-3, f"{what}: fused vs two-kernel |dO| {do} |dLSE| {dl}"


CASES = [
    # B, T, H, Hkv, d, N, dist, tree, splits
    (1, 64, 32, 8, 128, 3000, "V1", "beam", 0),       # CTA pairs (tree pass in the fused merge)
    (1, 64, 32, 8, 128, 4000, "V1", "beam", 64),      # pairs, 64 splits: a unit of 128 CTAs
    (1, 64, 8, 8, 128, 2500, "V2", "beam", 0),        # MHA single CTAs (fused tree tiles)
    (2, 64, 10, 2, 128, 1500, "V1", "beam", 0),       # G = 5: three row groups
    (4, 64, 40, 8, 128, 2048, "V1", "beam", 3),       # QwQ-like: 288 CTAs, two waves
    (1, 128, 32, 8, 128, 1280, "V1", "beam", 0),      # T = 128: two pair groups
    (1, 256, 8, 2, 128, 600, "V1", "beam", 2),        # T = 256: four pair groups, 4 rows per warp
    (2, 17, 4, 1, 64, 1100, "V1", "star", 0),         # d = 64
    (1, 30, 6, 2, 128, 900, "V0", "random", 7),       # G = 3 (Q staged by loads)
    (1, 1, 4, 4, 128, 1, "V1", "chain", 0),           # single key, single node
]


def _ids(c):
    return "B{}T{}H{}kv{}d{}N{}-{}-{}-s{}".format(*c)


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_fused_merge_vs_oracle_and_two_kernel(cuda_device, case):
    B, T, H, Hkv, d, N, dist, tree, splits = case
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist=dist, seed=41, tree=tree)
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    m_dev = torch.from_numpy(mask).to(cuda_device)
    shape = hta.make_shape(x["q"], k_cache=x["kc"], k_tree=x["kt"], num_splits=splits)
    ws = hta.new_workspace(shape, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)

    def run():
        return hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], m_dev, cache_seqlens=x["sl"], ws=ws,
                               num_splits=splits)

    fused, two = _both(run)
    compare(*fused, o_ref, l_ref, "bf16", f"fused {case}")
    compare(*two, o_ref, l_ref, "bf16", f"two-kernel {case}")
    _close(fused, two, str(case))
    assert int(_ctr_block(ws, shape).abs().sum()) == 0, "unit counters not re-armed / error word set"


@pytest.mark.parametrize("splits", [0, 5])
def test_fused_merge_empty_splits_and_garbage(cuda_device, splits):
    """Short and zero cache_seqlens: whole splits are empty (their CTAs only write sentinels, still
    arrive and take rows); NaN past the lengths never reaches the result."""
    sl = torch.tensor([1000, 0, 129, 1], dtype=torch.int32)
    for (H, Hkv) in ((8, 2), (32, 8)):
        w = make_workload(4, 64, H, Hkv, 128, 1024, "bf16", dist="V1", seed=5, tree="random", seqlens=sl,
                          garbage_tail=True)
        mask = oracle_masks(w)
        x = to_dev(w, cuda_device)
        shape = hta.make_shape(x["q"], k_cache=x["kc"], k_tree=x["kt"], num_splits=splits)
        ws = hta.new_workspace(shape, cuda_device)
        o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
        fused, two = _both(lambda: hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"],
                                                   torch.from_numpy(mask).to(cuda_device), cache_seqlens=x["sl"],
                                                   ws=ws, num_splits=splits))
        compare(*fused, o_ref, l_ref, "bf16", f"fused seqlens H={H}")
        _close(fused, two, f"seqlens H={H}")
        assert int(_ctr_block(ws, shape).abs().sum()) == 0


def test_fused_merge_forward_tree_and_paged(cuda_device):
    """hta_forward_tree (visibility from the parent array, walked in the fused merge's tree pass)
    and hta_forward_paged (same kernel over a page pool) through the fused merge."""
    w = make_workload(2, 64, 32, 8, 128, 2000, "bf16", dist="V1", seed=3, tree="beam")
    x = to_dev(w, cuda_device)
    par = torch.stack([tree_parents(k, 64, seed=b) for b, k in enumerate(("beam", "random"))])
    masks = np.stack([oracle.tree_mask(par[b]) for b in range(2)])
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, masks)
    p_dev = par.to(cuda_device)
    fused, two = _both(lambda: hta.hta_forward_tree(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], p_dev))
    compare(*fused, o_ref, l_ref, "bf16", "forward_tree fused")
    _close(fused, two, "forward_tree")
    # paged: 16-key pages of both batch entries shuffled in one pool
    page = 16
    n_pages = 2000 // page + 1
    perm = torch.randperm(2 * n_pages, generator=torch.Generator().manual_seed(0))
    kp = torch.zeros(2 * n_pages, page, 8, 128, dtype=torch.bfloat16)
    vp = torch.zeros_like(kp)
    bt = perm.view(2, n_pages).to(torch.int32)
    for b in range(2):
        for j in range(n_pages):
            lo, hi = j * page, min((j + 1) * page, 2000)
            if lo < hi:
                kp[bt[b, j], :hi - lo] = w.k_cache[b, lo:hi]
                vp[bt[b, j], :hi - lo] = w.v_cache[b, lo:hi]
    m_dev = torch.from_numpy(masks).to(cuda_device)
    fused, two = _both(lambda: hta.hta_forward_paged(x["q"], kp.to(cuda_device), vp.to(cuda_device),
                                                     bt.to(cuda_device), x["kt"], x["vt"], m_dev,
                                                     cache_seqlens=x["sl"]))
    compare(*fused, o_ref, l_ref, "bf16", "paged fused")
    _close(fused, two, "paged")


def test_fused_merge_graph_replays_bit_identical(cuda_device):
    """Captured once, replayed five times: every replay re-arms the counters and gives the eager
    result bit for bit."""
    w = make_workload(1, 64, 32, 8, 128, 5000, "bf16", dist="V1", seed=23, tree="beam")
    x = to_dev(w, cuda_device)
    m_dev = torch.from_numpy(oracle_masks(w)).to(cuda_device)
    shape = hta.make_shape(x["q"], k_cache=x["kc"], k_tree=x["kt"])
    ws = hta.new_workspace(shape, cuda_device)
    o = torch.empty_like(x["q"])
    lse = torch.empty(1, 32, 64, dtype=torch.float32, device=cuda_device)

    def step():
        hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], m_dev, o=o, lse_out=lse, ws=ws)

    step()
    torch.cuda.synchronize()
    ref_o, ref_l = o.clone(), lse.clone()
    s = torch.cuda.Stream(device=cuda_device)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(5):
        o.zero_()
        lse.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(o, ref_o) and torch.equal(lse, ref_l)
    assert int(_ctr_block(ws, shape).abs().sum()) == 0


def test_workspace_without_counter_room_uses_two_kernels(cuda_device):
    """A workspace holding only the partials (the pre-fusion size) still works: the split combine
    then runs as a second kernel."""
    w = make_workload(1, 64, 32, 8, 128, 3000, "bf16", dist="V1", seed=13, tree="beam")
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    shape = hta.make_shape(x["q"], k_cache=x["kc"], k_tree=x["kt"])
    full = hta.workspace_size(shape, torch.cuda.get_device_properties(cuda_device).multi_processor_count)
    G, units = 4, 1 * 8 * 2
    small = full - ((2 * units + 1) * 4 + 15) // 16 * 16
    ws = torch.full((small,), 0xFF, dtype=torch.uint8, device=cuda_device)  # garbage, no counters
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                           ws=ws)
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", "small workspace")
