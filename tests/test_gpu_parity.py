"""GPU parity: every ABI entry point vs the fp64 oracle on the same seeded inputs.

Sizes span several 128-key tiles with a ragged tail, several 128-row tiles (GQA row packing),
forced split counts, both dtypes, the three value distributions, and the edge cases (empty
prefix, garbage beyond cache_seqlens, T = 1, all-masked rows).  Full-size BASELINE configs are
checked on sampled rows in tests/test_gpu_configs.py.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload, random_mask, tree_parents
from workloads.generators import named_generator

from gpu_util import compare, oracle_masks, to_dev

pytestmark = pytest.mark.gpu

CASES = [
    # B, T, H, Hkv, d, N, dtype, dist, tree
    (1, 8, 1, 1, 64, 256, "fp32", "V1", "heap_binary"),      # BASELINE configs[0] (toy)
    (2, 13, 8, 2, 128, 1000, "bf16", "V1", "random"),        # G=4, M=52, ragged tail
    (1, 64, 32, 8, 128, 3000, "bf16", "V1", "beam"),         # M=256: two row tiles per CTA
    (1, 64, 8, 8, 128, 2500, "bf16", "V2", "beam"),          # MHA, M=64 (LongChat-like rows)
    (2, 64, 10, 2, 128, 1500, "bf16", "V1", "beam"),         # G=5, M=320: three row groups
    (1, 40, 8, 2, 128, 777, "bf16", "V0", "chain"),          # M=160: second tile partly used
    (1, 80, 10, 2, 128, 640, "bf16", "V1", "random_forest"),  # M=400: second group half used
    (2, 17, 4, 1, 64, 1100, "bf16", "V1", "star"),           # d=64
    (1, 128, 32, 8, 128, 1280, "bf16", "V1", "beam"),        # T=128, M=512
    (3, 5, 6, 3, 128, 300, "fp32", "V2", "random"),          # fp32 GQA
    (1, 1, 4, 4, 128, 1, "bf16", "V1", "chain"),             # single key, single node
    (2, 7, 4, 2, 64, 129, "fp32", "V0", "roots"),            # fp32 d=64, self-only tree
    (1, 30, 6, 2, 128, 900, "bf16", "V1", "random"),         # G=3: Q staged by loads, one CTA
    (2, 9, 6, 2, 64, 700, "bf16", "V2", "beam"),             # G=3, d=64
    (1, 256, 8, 2, 128, 600, "bf16", "V1", "beam"),          # T=256 (the maximum), M=1024: 4 pair groups
    (1, 64, 32, 1, 128, 1000, "bf16", "V1", "beam"),         # MQA (H_kv=1, G=32), M=2048
    (2, 33, 8, 8, 64, 2049, "bf16", "V2", "random"),         # MHA d=64, N just past a 192-key tile
]


def _ids(c):
    return "B{}T{}H{}kv{}d{}N{}-{}-{}-{}".format(*c)


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_forward_and_parts_vs_oracle(cuda_device, case):
    B, T, H, Hkv, d, N, dtype, dist, tree = case
    w = make_workload(B, T, H, Hkv, d, N, dtype, dist=dist, seed=7, tree=tree)
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    m_dev = torch.from_numpy(mask).to(cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    oc_ref, lc_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, part="cache")
    ot_ref, lt_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, part="tree")

    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], m_dev, cache_seqlens=x["sl"])
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, dtype, "forward")
    oc, lc = hta.hta_prefix_attn(x["q"], x["kc"], x["vc"])
    torch.cuda.synchronize()
    compare(oc, lc, oc_ref, lc_ref, dtype, "prefix")
    ot, lt = hta.hta_tree_attn(x["q"], x["kt"], x["vt"], m_dev)
    torch.cuda.synchronize()
    compare(ot, lt, ot_ref, lt_ref, dtype, "tree")
    # merging the two ABI partials with hta_merge_lse reproduces the forward
    om, lm = hta.hta_merge_lse(torch.stack([oc, ot]), torch.stack([lc, lt]), dtype=w.torch_dtype, H_kv=Hkv)
    torch.cuda.synchronize()
    compare(om, lm, o_ref, l_ref, dtype, "merge")


@pytest.mark.parametrize("splits", [1, 2, 3, 7, 64])
def test_forced_split_counts(cuda_device, splits):
    w = make_workload(1, 64, 32, 8, 128, 4000, "bf16", dist="V1", seed=11, tree="beam")
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                           num_splits=splits)
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", f"splits={splits}")


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_seqlens_with_nan_garbage_tail(cuda_device, dtype):
    """Z13: rows >= cache_seqlens[b] hold NaN and must never reach the softmax; an empty
    prefix (seqlen 0) gives the tree-only result."""
    sl = torch.tensor([1000, 0, 129, 1], dtype=torch.int32)
    w = make_workload(4, 9, 8, 2, 128, 1024, dtype, dist="V1", seed=5, tree="random", seqlens=sl,
                      garbage_tail=True)
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    for splits in (0, 5):
        o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                               cache_seqlens=x["sl"], num_splits=splits)
        torch.cuda.synchronize()
        compare(o, l, o_ref, l_ref, dtype, f"seqlens splits={splits}")
    oc_ref, lc_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens,
                                      part="cache")
    oc, lc = hta.hta_prefix_attn(x["q"], x["kc"], x["vc"], cache_seqlens=x["sl"])
    torch.cuda.synchronize()
    compare(oc, lc, oc_ref, lc_ref, dtype, "prefix seqlens")   # batch 1 is the sentinel


def test_arbitrary_masks_and_empty_rows(cuda_device):
    """The tree pass accepts any 0/1 pattern; an all-zero row is the sentinel, and the forward
    then equals the prefix part."""
    w = make_workload(2, 70, 4, 2, 128, 300, "bf16", dist="V1", seed=9, tree="random")
    mask = random_mask(2, 70, 0.3, seed=3).numpy()
    mask[0, 5] = 0
    mask[1, 69] = 0
    x = to_dev(w, cuda_device)
    m_dev = torch.from_numpy(mask).to(cuda_device)
    ot_ref, lt_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, part="tree")
    ot, lt = hta.hta_tree_attn(x["q"], x["kt"], x["vt"], m_dev)
    torch.cuda.synchronize()
    compare(ot, lt, ot_ref, lt_ref, "bf16", "tree random mask")
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], m_dev)
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", "forward random mask")


def test_shared_mask_batch_stride_zero(cuda_device):
    w = make_workload(3, 16, 8, 2, 128, 500, "bf16", dist="V1", seed=12, tree="heap_binary")
    m1 = oracle.tree_mask(w.parents[0])
    mask = np.stack([m1] * 3)
    x = to_dev(w, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(m1).to(cuda_device))
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", "shared mask")


def test_strided_layouts(cuda_device):
    """KV in [B, H_kv, N, d] memory order and q/o as a slice of a wider tensor (strides)."""
    w = make_workload(2, 12, 8, 2, 128, 700, "bf16", dist="V1", seed=13, tree="random")
    mask = oracle_masks(w)
    dev = cuda_device
    kc = w.k_cache.permute(0, 2, 1, 3).contiguous().to(dev).permute(0, 2, 1, 3)   # strides of [B,Hkv,N,d]
    vc = w.v_cache.permute(0, 2, 1, 3).contiguous().to(dev).permute(0, 2, 1, 3)
    qbig = torch.zeros(2, 12, 16, 128, dtype=torch.bfloat16, device=dev)
    qbig[:, :, 4:12] = w.q.to(dev)
    q = qbig[:, :, 4:12]
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    o, l = hta.hta_forward(q, kc, vc, w.k_tree.to(dev), w.v_tree.to(dev), torch.from_numpy(mask).to(dev))
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", "strided")


def test_simulated_sequence_sharding(cuda_device):
    """a5 on one GPU: P contiguous KV slices through hta_prefix_attn (strided views), the tree
    part through hta_tree_attn, all P+1 partials through hta_merge_lse == one-shot oracle."""
    w = make_workload(1, 64, 32, 8, 128, 4096, "bf16", dist="V1", seed=14, tree="beam")
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    for P in (2, 4, 8):
        parts_o, parts_l = [], []
        for r in range(P):
            lo, hi = hta.shard_bounds(4096, P, r)
            oc, lc = hta.hta_prefix_attn(x["q"], x["kc"][:, lo:hi], x["vc"][:, lo:hi])
            parts_o.append(oc)
            parts_l.append(lc)
        ot, lt = hta.hta_tree_attn(x["q"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device))
        parts_o.append(ot)
        parts_l.append(lt)
        o, l = hta.hta_merge_lse(torch.stack(parts_o), torch.stack(parts_l), dtype=torch.bfloat16, H_kv=8)
        torch.cuda.synchronize()
        compare(o, l, o_ref, l_ref, "bf16", f"sharded P={P}")


def test_device_mask_builder_bit_exact(cuda_device):
    for seed in range(30):
        T = [1, 8, 64, 128, 256][seed % 5]
        kind = ["random", "random_forest", "beam", "chain", "heap_binary", "star"][seed % 6]
        par = tree_parents(kind, T, seed=seed)
        m = hta.hta_build_tree_mask(par.to(cuda_device))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(m.cpu().numpy(), oracle.tree_mask(par))
    bad = torch.tensor([-1, 0, 5, 1], dtype=torch.int32, device=cuda_device)
    m = hta.hta_build_tree_mask(bad).cpu().numpy()
    assert m[2].sum() == 0 and m[3].tolist() == [1, 1, 0, 1]


def test_device_accept_bit_exact(cuda_device):
    from workloads import accept_tokens
    for seed in range(200):
        T = [1, 3, 8, 17, 64, 128, 256][seed % 7]
        kind = ["random", "random_forest", "beam", "chain", "star"][seed % 5]
        par = tree_parents(kind, T, seed=seed)
        draft, tgt, ctx = accept_tokens(par, seed, vocab=4, p_match=0.8, distinct_siblings=(seed % 2 == 0))
        for root in ((0, -1) if kind != "random_forest" else (-1,)):
            path, plen, bonus = hta.hta_accept_greedy(par.to(cuda_device), draft.to(cuda_device),
                                                      tgt.to(cuda_device), root=root, context_argmax=ctx)
            torch.cuda.synchronize()
            want_path, want_bonus = oracle.accept_greedy(par, draft, tgt, root=root, context_argmax=ctx)
            n = int(plen.item())
            assert path[:n].cpu().tolist() == want_path and int(bonus.item()) == want_bonus, (seed, root)


def test_tree_step_bit_exact(cuda_device):
    """hta_tree_step (a0 + a6 in one launch): the mask equals the recursive-ancestor oracle and
    the path / bonus equal the brute-force accept oracle, including invalid parent arrays and
    every root choice on small trees (duplicate sibling tokens on odd seeds)."""
    from workloads import accept_tokens
    for seed in range(240):
        T = [1, 2, 5, 8, 17, 33, 64, 128, 200, 256][seed % 10]
        kind = ["random", "random_forest", "beam", "chain", "star", "heap_binary"][seed % 6]
        par = tree_parents(kind, T, seed=seed)
        draft, tgt, ctx = accept_tokens(par, seed, vocab=3, p_match=0.85, distinct_siblings=(seed % 2 == 0))
        roots = (-1,) if kind == "random_forest" else ((0, -1) + ((T // 2,) if T > 2 else ()))
        for root in roots:
            m, path, plen, bonus = hta.hta_tree_step(par.to(cuda_device), draft.to(cuda_device), tgt.to(cuda_device),
                                                     root=root, context_argmax=ctx)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(m.cpu().numpy(), oracle.tree_mask(par))
            want_path, want_bonus = oracle.accept_greedy(par, draft, tgt, root=root, context_argmax=ctx)
            n = int(plen.item())
            assert path[:n].cpu().tolist() == want_path and int(bonus.item()) == want_bonus, (seed, root)
    # invalid parents: path_len = -1, the offending row is all zero
    bad = torch.tensor([-1, 0, 5, 1], dtype=torch.int32)
    d0 = torch.zeros(4, dtype=torch.int32)
    m, path, plen, bonus = hta.hta_tree_step(bad.to(cuda_device), d0.to(cuda_device), d0.to(cuda_device), root=0)
    torch.cuda.synchronize()
    assert int(plen.item()) == -1 and int(m[2].sum().item()) == 0 and int(m[3].sum().item()) == 3


def test_deterministic(cuda_device):
    w = make_workload(1, 64, 32, 8, 128, 5000, "bf16", dist="V1", seed=15, tree="beam")
    mask = torch.from_numpy(oracle_masks(w)).to(cuda_device)
    x = to_dev(w, cuda_device)
    o1, l1 = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask)
    o2, l2 = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_step_in_cuda_graph_matches_eager(cuda_device):
    """bench.py replays the step (mask -> forward, accept on a forked stream) from a CUDA graph;
    the replay (with programmatic dependent launches as graph edges) must give the eager results."""
    from workloads import accept_tokens
    w = make_workload(1, 64, 32, 8, 128, 3000, "bf16", dist="V1", seed=17, tree="beam")
    x = to_dev(w, cuda_device)
    par = w.parents[0].to(cuda_device)
    dr, tg, ctx = accept_tokens(w.parents[0], seed=1, vocab=1000, p_match=0.8)
    dr, tg = dr.to(cuda_device), tg.to(cuda_device)
    mask = torch.empty(64, 64, dtype=torch.uint8, device=cuda_device)
    o = torch.empty_like(x["q"])
    lse = torch.empty(1, 32, 64, dtype=torch.float32, device=cuda_device)
    path = torch.empty(64, dtype=torch.int32, device=cuda_device)
    plen = torch.empty(1, dtype=torch.int32, device=cuda_device)
    bonus = torch.empty(1, dtype=torch.int32, device=cuda_device)
    wsb = hta.new_workspace(hta.make_shape(x["q"], k_cache=x["kc"], k_tree=x["kt"]), cuda_device)
    side = torch.cuda.Stream(device=cuda_device)

    def step():
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            hta.hta_accept_greedy(par, dr, tg, root=0, path=path, path_len=plen, bonus=bonus)
        hta.hta_build_tree_mask(par, mask)
        hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask, cache_seqlens=x["sl"], o=o, lse_out=lse,
                        ws=wsb)
        cur.wait_stream(side)

    for t in (o, lse, path, plen, bonus):  # (path is written up to path_len only)
        t.zero_()
    step()
    torch.cuda.synchronize()
    ref = [t.clone() for t in (o, lse, path, plen, bonus)]
    for t in (o, lse, path, plen, bonus):
        t.zero_()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(device=cuda_device)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for t in (o, lse, path, plen, bonus):
        t.zero_()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for name, a, b in zip(("o", "lse", "path", "path_len", "bonus"), (o, lse, path, plen, bonus), ref):
        assert torch.equal(a, b), f"{name}: max |diff| {(a.float() - b.float()).abs().max().item()}"


@pytest.mark.parametrize("key", [192 + 2, 192 + 96 + 17, 192 + 9, 384 + 50, 3])
@pytest.mark.parametrize("d,dtype", [(128, "bf16"), (64, "bf16"), (128, "fp32")])
def test_logit_jump_past_exp_range(cuda_device, key, d, dtype):
    """One prefix key whose logit exceeds the running max of the earlier tiles by ~150 (natural
    units, 2^216 in P): the speculative exponentials overflow and the tile is redone with the
    true max (prefix_tc.cu).  The key positions put the jump into polynomial and
    MUFU exp slots of both column halves, in tiles 0-2 of one split (Z4 max-shifting: the result
    must still equal the fp64 softmax)."""
    B, T, H, Hkv, N = 1, 4, 4, 1, 576
    gen = named_generator(11, f"jump:{key}:{d}")
    u = torch.randn(d, generator=gen)
    u = u / u.norm()
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q = (40.0 * u + 0.5 * torch.randn(B, T, H, d, generator=gen)).to(tdt)
    kc = torch.randn(B, N, Hkv, d, generator=gen)
    kc[:, key, :, :] = 42.5 * u + 0.1 * kc[:, key, :, :]  # logit ~150 (d=128) / ~205 (d=64)
    kc = kc.to(tdt)
    vc = torch.randn(B, N, Hkv, d, generator=gen).to(tdt)
    kt = torch.zeros(B, T, Hkv, d, dtype=tdt)
    mask = np.ones((B, T, T), np.uint8)
    oc_ref, lc_ref = oracle.attention(q, kc, vc, kt, kt, mask, part="cache")
    for splits in (1, 2):
        oc, lc = hta.hta_prefix_attn(q.to(cuda_device), kc.to(cuda_device), vc.to(cuda_device), num_splits=splits)
        torch.cuda.synchronize()
        compare(oc, lc, oc_ref, lc_ref, dtype, f"prefix (S={splits})")


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_tree_logit_far_above_prefix(cuda_device, dtype):
    """A tree key whose logit exceeds every prefix logit by ~150 (and rows whose tree part is
    far BELOW the prefix): the LSE merge must weight the parts by exp of LSE
    differences far outside the fp32 exp range without overflow (Z4)."""
    B, T, H, Hkv, d, N = 2, 6, 4, 2, 128, 700
    gen = named_generator(12, f"treejump:{dtype}")
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    u = torch.randn(d, generator=gen)
    u = u / u.norm()
    q = (40.0 * u + 0.5 * torch.randn(B, T, H, d, generator=gen)).to(tdt)
    kc = torch.randn(B, N, Hkv, d, generator=gen)
    kt = torch.randn(B, T, Hkv, d, generator=gen)
    kt[0, 2] = 42.5 * u          # batch 0: tree node 2 dominates the rows that see it
    kc[1, 123] = 42.5 * u        # batch 1: a prefix key dominates, the tree part is ~150 below
    q, kc, kt = q.to(tdt), kc.to(tdt), kt.to(tdt)
    vc = torch.randn(B, N, Hkv, d, generator=gen).to(tdt)
    vt = torch.randn(B, T, Hkv, d, generator=gen).to(tdt)
    parents = torch.stack([torch.tensor([-1, 0, 0, 1, 2, 2], dtype=torch.int32)] * B)
    mask = np.stack([oracle.tree_mask(parents[b]) for b in range(B)])
    o_ref, l_ref = oracle.attention(q, kc, vc, kt, vt, mask)
    x = [t.to(cuda_device) for t in (q, kc, vc, kt, vt)]
    o, l = hta.hta_forward(*x, torch.from_numpy(mask).to(cuda_device))
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, dtype, "forward")


def test_max_seqlen_hint_plans_by_filled_length(cuda_device):
    """A preallocated cache much longer than its filled length: hta_shape_t.max_seqlen plans the
    split-KV schedule over the filled length; the result is exact whether the bound holds (1200
    >= every length) or is violated (600 < 1000: the last split runs to each entry's length)."""
    sl = torch.tensor([1000, 37], dtype=torch.int32)
    w = make_workload(2, 16, 8, 2, 128, 16384, "bf16", dist="V1", seed=21, tree="beam", seqlens=sl,
                      garbage_tail=True)
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    for hint in (1200, 600, 0):
        o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                               cache_seqlens=x["sl"], max_seqlen=hint)
        torch.cuda.synchronize()
        compare(o, l, o_ref, l_ref, "bf16", f"max_seqlen={hint}")


def test_forward_ex_tree_inputs_late(cuda_device):
    """hta_forward_ex: k_tree / v_tree / mask produced on another stream after the call is
    enqueued; only the tree/merge kernel waits for them (the event; the tree pass then runs in
    that kernel instead of the prefix kernel), and the result matches the oracle as
    hta_forward's does."""
    w = make_workload(1, 64, 32, 8, 128, 3000, "bf16", dist="V1", seed=19, tree="beam")
    mask_h = torch.from_numpy(oracle_masks(w)[0])
    x = to_dev(w, cuda_device)
    o_ref, l_ref = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask_h.to(cuda_device))
    kt = torch.zeros_like(x["kt"])
    vt = torch.zeros_like(x["vt"])
    m = torch.zeros(64, 64, dtype=torch.uint8, device=cuda_device)
    side = torch.cuda.Stream()
    ready = torch.cuda.Event()
    torch.cuda.synchronize()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        torch.cuda._sleep(2_000_000)  # the tree inputs land well after the prefix pass started
        kt.copy_(x["kt"])
        vt.copy_(x["vt"])
        m.copy_(mask_h.to(cuda_device))
        ready.record()
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], kt, vt, m, tree_ready=ready)
    torch.cuda.synchronize()
    oo, lo = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, oracle_masks(w))
    compare(o_ref, l_ref, oo, lo, "bf16", "forward (fused tree pass)")
    compare(o, l, oo, lo, "bf16", "forward_ex (tree inputs late)")


@pytest.mark.parametrize("case", [
    # B, T, H, Hkv, d, N, seqlens, num_splits: single-CTA row groups (the fused tree pass)
    (2, 200, 2, 2, 64, 700, (700, 0), 0),       # two tree tiles; an empty cache
    (3, 64, 8, 8, 128, 1000, (1000, 1, 129), 0),  # MHA (LongChat rows); 1-key and 129-key caches
    (2, 64, 10, 2, 128, 900, (900, 300), 7),    # G = 5, forced splits: the last split holds only tree
    (1, 17, 3, 1, 128, 16, (0,), 0),            # an empty cache: the tree tile alone
])
def test_fused_tree_pass_edge_cases(cuda_device, case):
    """hta_forward runs the tree pass inside the prefix kernel for single-CTA row groups (tree
    tiles appended to each unit's last split, masked in TMEM).  Arbitrary masks with empty rows,
    caches shorter than a tile or empty, two tree tiles (T > 128) and a last split holding only
    the tree tile all match the oracle; an all-zero mask row over an empty cache is the sentinel
    (O = 0, LSE = -inf)."""
    B, T, H, Hkv, d, N, sl, ns = case
    seqlens = torch.tensor(sl, dtype=torch.int32)
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist="V1", seed=41, tree="random", seqlens=seqlens,
                      garbage_tail=True)
    mask = random_mask(B, T, 0.35, seed=7).numpy()
    mask[0, 3] = 0
    mask[-1, T - 1] = 0
    x = to_dev(w, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                           cache_seqlens=x["sl"], num_splits=ns)
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", f"fused tree pass {case}")


@pytest.mark.parametrize("case", [
    # B, T, H, Hkv, d, N, tree kinds per batch entry (one shared tree when a single kind)
    (1, 64, 32, 8, 128, 3000, ("beam",)),                 # CTA pairs: the tree pass walks in the tree/merge kernel
    (2, 64, 8, 8, 128, 2000, ("random", "chain")),        # MHA single CTAs: the walk in the prefix kernel
    (2, 200, 4, 2, 64, 900, ("random_forest", "star")),   # two tree tiles, forests (several roots)
    (1, 256, 16, 4, 128, 700, ("chain",)),                # T = 256, depth 255
    (3, 30, 10, 2, 128, 500, ("heap_binary", "roots", "random")),  # G = 5
    (1, 8, 1, 1, 64, 256, ("heap_binary",), "fp32"),      # the toy config (fp32 SIMT prefix)
])
def test_forward_tree_from_parents(cuda_device, case):
    """hta_forward_tree derives each row's visible tree keys from the parent array inside the
    kernels (Z4).  Its result is bit-identical to hta_forward over the mask hta_build_tree_mask
    writes, and matches the oracle over the oracle's tree mask."""
    B, T, H, Hkv, d, N, kinds = case[:7]
    dt = case[7] if len(case) > 7 else "bf16"
    w = make_workload(B, T, H, Hkv, d, N, dt, dist="V1", seed=29, tree="beam")
    par = torch.stack([tree_parents(kinds[b % len(kinds)], T, seed=b) for b in range(B)])
    shared = len(kinds) == 1
    x = to_dev(w, cuda_device)
    p_dev = par[0].to(cuda_device) if shared else par.to(cuda_device)
    masks = np.stack([oracle.tree_mask(par[0 if shared else b]) for b in range(B)])
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, masks)
    o, l = hta.hta_forward_tree(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], p_dev)
    m_dev = torch.stack([hta.hta_build_tree_mask(par[0 if shared else b].to(cuda_device)) for b in range(B)])
    om, lm = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], m_dev)
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, dt, f"forward_tree {case}")
    assert torch.equal(o, om) and torch.equal(l, lm), "hta_forward_tree differs from hta_forward over the built mask"


def test_forward_tree_invalid_parents_hide_rows(cuda_device):
    """An invalid parent entry hides every row whose chain meets it, exactly as the all-zero rows
    hta_build_tree_mask writes for it (pairs and single CTAs)."""
    for (H, Hkv) in ((32, 8), (8, 8)):
        w = make_workload(1, 64, H, Hkv, 128, 1500, "bf16", dist="V1", seed=31, tree="beam")
        par = tree_parents("random", 64, seed=4).clone()
        par[10] = 10        # self-parent
        par[40] = 57        # a later node
        par[50] = -3        # below -1
        x = to_dev(w, cuda_device)
        p_dev = par.to(cuda_device)
        o, l = hta.hta_forward_tree(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], p_dev)
        m_dev = hta.hta_build_tree_mask(p_dev)
        om, lm = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], m_dev)
        torch.cuda.synchronize()
        assert m_dev.sum(1).eq(0).any(), "the invalid entries must hide some rows"
        assert torch.equal(o, om) and torch.equal(l, lm)
