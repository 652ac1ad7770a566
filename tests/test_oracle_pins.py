"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test ties the oracle to a closed form, a library routine (torch SDPA in float64), an
exact identity of the paper (Appendix C), a hand-worked fixture under tests/golden/, or
brute force.  A plausible bug in oracle/ -- a dropped term, a wrong sign, a transposed
operand, a wrong GQA head map, a wrong scale, a missing max-shift -- fails one of these.
"""
import itertools
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from workloads import make_workload, tree_parents
from workloads.generators import named_generator

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, seed, name, scale=1.0):
    return (torch.randn(*shape, generator=named_generator(seed, name)) * scale).double()


def sdpa64(q, k, v, allow, scale=None):
    """torch SDPA in float64.  q [Lq,d], k/v [Lk,d], allow bool [Lq,Lk].  The scale defaults
    to 1/sqrt(d) rounded to float32, the value the kernels receive (reading Z2)."""
    if scale is None:
        scale = float(np.float32(1 / math.sqrt(q.shape[-1])))
    o = F.scaled_dot_product_attention(q[None, None], k[None, None], v[None, None],
                                       attn_mask=allow[None, None], scale=scale)
    return o[0, 0]


def lse64(q, k, allow, scale):
    z = (q @ k.T) * scale
    z = z.masked_fill(~allow, float("-inf"))
    return torch.logsumexp(z, dim=-1)


def oracle_inputs(B, T, H, Hkv, d, N, seed, q_scale=1.0):
    q = _rand((B, T, H, d), seed, "q", q_scale).float()
    kc = _rand((B, N, Hkv, d), seed, "kc").float()
    vc = _rand((B, N, Hkv, d), seed, "vc").float()
    kt = _rand((B, T, Hkv, d), seed, "kt").float()
    vt = _rand((B, T, Hkv, d), seed, "vt").float()
    return q, kc, vc, kt, vt


# ----------------------------------------------------------------------- closed forms

def test_zero_query_gives_mean_and_log_n():
    """q = 0 -> every logit is 0: O = mean(V_cache[:n]), LSE = ln n (cache part)."""
    B, T, H, Hkv, d, N = 2, 3, 4, 2, 16, 37
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 1)
    q.zero_()
    seqlens = torch.tensor([37, 11], dtype=torch.int32)
    mask = np.ones((B, T, T), np.uint8)
    o, lse = oracle.attention(q, kc, vc, kt, vt, mask, seqlens=seqlens, part="cache")
    for b in range(B):
        n = int(seqlens[b])
        for h in range(H):
            g = h // (H // Hkv)
            want = vc[b, :n, g].double().mean(0).numpy()
            for t in range(T):
                np.testing.assert_allclose(o[b, t, h], want, rtol=0, atol=1e-13)
                assert abs(lse[b, h, t] - math.log(n)) < 1e-13


def test_single_key_closed_form():
    """n = 1 -> O = v_0 and LSE = scale * q.k_0."""
    B, T, H, Hkv, d, N = 1, 2, 2, 1, 32, 1
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 2)
    o, lse = oracle.attention(q, kc, vc, kt, vt, np.ones((B, T, T), np.uint8), part="cache", scale=0.25)
    for t in range(T):
        for h in range(H):
            np.testing.assert_array_equal(o[0, t, h], vc[0, 0, 0].double().numpy())
            want = 0.25 * float(np.dot(q[0, t, h].double().numpy(), kc[0, 0, 0].double().numpy()))
            assert abs(lse[0, h, t] - want) < 1e-12


def test_equal_rows_closed_forms():
    """All V rows equal -> O = v.  All K rows equal -> LSE = scale q.k + ln n, O = mean V."""
    B, T, H, Hkv, d, N = 1, 2, 2, 2, 8, 9
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 3)
    vc_eq = vc.clone()
    vc_eq[:] = vc[:, :1]
    o, _ = oracle.attention(q, kc, vc_eq, kt, vt, np.ones((B, T, T), np.uint8), part="cache")
    for h in range(H):
        np.testing.assert_allclose(o[0, :, h], np.broadcast_to(vc[0, 0, h].double().numpy(), (T, d)),
                                   rtol=1e-14, atol=1e-14)
    kc_eq = kc.clone()
    kc_eq[:] = kc[:, :1]
    o, lse = oracle.attention(q, kc_eq, vc, kt, vt, np.ones((B, T, T), np.uint8), part="cache")
    s = float(np.float32(1 / math.sqrt(d)))
    for t in range(T):
        for h in range(H):
            want = s * float(np.dot(q[0, t, h].double().numpy(), kc[0, 0, h].double().numpy())) + math.log(N)
            assert abs(lse[0, h, t] - want) < 1e-12
            np.testing.assert_allclose(o[0, t, h], vc[0, :, h].double().mean(0).numpy(), atol=1e-13)


def test_self_only_mask_tree_part():
    """Star of roots (self-only mask) -> O_i = v_i, LSE_i = scale q_i.k_i."""
    B, T, H, Hkv, d, N = 1, 5, 4, 2, 16, 3
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 4)
    mask = np.eye(T, dtype=np.uint8)[None]
    o, lse = oracle.attention(q, kc, vc, kt, vt, mask, part="tree")
    s = float(np.float32(1 / math.sqrt(d)))
    for t in range(T):
        for h in range(H):
            g = h // 2
            np.testing.assert_array_equal(o[0, t, h], vt[0, t, g].double().numpy())
            assert abs(lse[0, h, t] - s * float(np.dot(q[0, t, h].double().numpy(),
                                                        kt[0, t, g].double().numpy()))) < 1e-12


def test_empty_parts_are_sentinels():
    """n = 0 cache part and an all-zero mask row give (O = 0, LSE = -inf) (Z10)."""
    B, T, H, Hkv, d, N = 1, 3, 2, 1, 8, 4
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 5)
    o, lse = oracle.attention(q, kc, vc, kt, vt, np.ones((B, T, T), np.uint8),
                              seqlens=torch.tensor([0], dtype=torch.int32), part="cache")
    assert np.all(o == 0) and np.all(np.isneginf(lse))
    mask = np.ones((B, T, T), np.uint8)
    mask[0, 1] = 0
    o, lse = oracle.attention(q, kc, vc, kt, vt, mask, part="tree")
    assert np.all(o[0, 1] == 0) and np.all(np.isneginf(lse[0, :, 1]))
    assert np.all(np.isfinite(lse[0, :, 0]))


# ----------------------------------------------------------------------- library routine

@pytest.mark.parametrize("T,G", [(1, 1), (6, 2), (9, 4)])
def test_chain_mask_is_causal_attention(T, G):
    """I1: a chain tree equals causal attention over [cache; tree], bottom-right aligned,
    computed by torch SDPA (float64) with GQA expanded by repeat_interleave (HF repeat_kv)."""
    B, Hkv, d, N = 2, 2, 32, 13
    H = Hkv * G
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 10 + T)
    mask = np.stack([oracle.tree_mask(tree_parents("chain", T))] * B)
    o, lse = oracle.attention(q, kc, vc, kt, vt, mask)
    L = N + T
    allow = torch.ones(T, L, dtype=torch.bool)
    for t in range(T):
        allow[t, N + t + 1:] = False   # query t sits at absolute position N + t
    for b in range(B):
        K = torch.cat([kc[b], kt[b]]).double().repeat_interleave(G, dim=1)   # [L, H, d]
        V = torch.cat([vc[b], vt[b]]).double().repeat_interleave(G, dim=1)
        for h in range(H):
            ref = sdpa64(q[b, :, h].double(), K[:, h], V[:, h], allow)
            np.testing.assert_allclose(o[b, :, h], ref.numpy(), rtol=1e-12, atol=1e-12)
            ref_lse = lse64(q[b, :, h].double(), K[:, h], allow, float(np.float32(1 / math.sqrt(d))))
            np.testing.assert_allclose(lse[b, h], ref_lse.numpy(), rtol=1e-12, atol=1e-12)


def test_single_node_is_decode_attention():
    """I2: T = 1 equals ordinary decode attention over n + 1 keys (SDPA, no mask)."""
    B, T, H, Hkv, d, N = 3, 1, 8, 2, 64, 50
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 20)
    seqlens = torch.tensor([50, 7, 0], dtype=torch.int32)
    o, _ = oracle.attention(q, kc, vc, kt, vt, np.ones((B, 1, 1), np.uint8), seqlens=seqlens)
    for b in range(B):
        n = int(seqlens[b])
        K = torch.cat([kc[b, :n], kt[b]]).double().repeat_interleave(H // Hkv, dim=1)
        V = torch.cat([vc[b, :n], vt[b]]).double().repeat_interleave(H // Hkv, dim=1)
        for h in range(H):
            ref = sdpa64(q[b, :, h].double(), K[:, h], V[:, h], torch.ones(1, n + 1, dtype=torch.bool))
            np.testing.assert_allclose(o[b, 0, h], ref[0].numpy(), rtol=1e-12, atol=1e-12)


def test_explicit_scale_and_gqa_head_map():
    """A non-default scale and G = 5 (QwQ-like 40q/8kv): compare with SDPA(scale=...)."""
    B, T, H, Hkv, d, N = 1, 4, 10, 2, 16, 21
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 21)
    mask = np.stack([oracle.tree_mask(tree_parents("heap_binary", T))])
    o, _ = oracle.attention(q, kc, vc, kt, vt, mask, scale=0.3)
    K = torch.cat([kc[0], kt[0]]).double().repeat_interleave(5, dim=1)
    V = torch.cat([vc[0], vt[0]]).double().repeat_interleave(5, dim=1)
    allow = torch.cat([torch.ones(T, N, dtype=torch.bool), torch.from_numpy(mask[0]).bool()], 1)
    for h in range(H):
        ref = F.scaled_dot_product_attention(q[0, :, h].double()[None, None], K[:, h][None, None],
                                             V[:, h][None, None], attn_mask=allow[None, None],
                                             scale=0.3)[0, 0]
        np.testing.assert_allclose(o[0, :, h], ref.numpy(), rtol=1e-12, atol=1e-12)


def test_brute_force_all_small_trees():
    """I4: every parent array with parents[i] in [-1, i) for T <= 4 (24 trees), N <= 3:
    row i equals unmasked SDPA over prefix + the node's root path (path linearisation)."""
    d, Hkv, H = 8, 1, 2
    for T in range(1, 5):
        for par in itertools.product(*[range(-1, i) for i in range(T)]):
            for N in (0, 3):
                q, kc, vc, kt, vt = oracle_inputs(1, T, H, Hkv, d, max(N, 1), 30 + T)
                mask = oracle.tree_mask(list(par))[None]
                o, _ = oracle.attention(q, kc, vc, kt, vt, mask,
                                        seqlens=torch.tensor([N], dtype=torch.int32))
                for i in range(T):
                    path = [i]
                    while par[path[-1]] >= 0:
                        path.append(par[path[-1]])
                    K = torch.cat([kc[0, :N, 0], kt[0, path, 0]]).double()
                    V = torch.cat([vc[0, :N, 0], vt[0, path, 0]]).double()
                    for h in range(H):
                        ref = sdpa64(q[0, i:i + 1, h].double(), K, V,
                                     torch.ones(1, K.shape[0], dtype=torch.bool))
                        np.testing.assert_allclose(o[0, i, h], ref[0].numpy(), rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------------- identities

def test_merge_identity_appendix_c_1000_cases():
    """I3 / PAPER.md:590-598 (Appendix C): merge(prefix part, tree part) equals one-shot
    attention over the union, within 1e-12, on 1000 random rows."""
    B, T, H, Hkv, d, N = 4, 10, 5, 5, 16, 33   # 4*10*5*... rows; loop seeds to reach 1000
    rows = 0
    seed = 100
    while rows < 1000:
        q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, seed, q_scale=3.0)
        parents = tree_parents("random_forest", T, seed=seed)
        mask = np.stack([oracle.tree_mask(parents)] * B)
        seqlens = torch.randint(0, N + 1, (B,), generator=named_generator(seed, "sl"), dtype=torch.int32)
        full = oracle.attention(q, kc, vc, kt, vt, mask, seqlens=seqlens)
        pc = oracle.attention(q, kc, vc, kt, vt, mask, seqlens=seqlens, part="cache")
        pt = oracle.attention(q, kc, vc, kt, vt, mask, seqlens=seqlens, part="tree")
        mo, ml = oracle.merge([(pc[0], pc[1].transpose(0, 2, 1)), (pt[0], pt[1].transpose(0, 2, 1))])
        np.testing.assert_allclose(mo, full[0], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(ml.transpose(0, 2, 1), full[1], rtol=1e-12, atol=1e-12)
        rows += B * T * H
        seed += 1


@pytest.mark.parametrize("P", [2, 3, 8])
def test_split_associativity(P):
    """A P-way split of the prefix + the tree part, merged, equals one-shot."""
    B, T, H, Hkv, d, N = 1, 7, 4, 2, 16, 50
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 40 + P, q_scale=2.0)
    mask = oracle.tree_mask(tree_parents("random", T, seed=P))[None]
    full = oracle.attention(q, kc, vc, kt, vt, mask)
    bounds = [N * r // P for r in range(P + 1)]
    parts = []
    for r in range(P):
        o, l = oracle.attention(q, kc, vc, kt, vt, mask, part="cache", cache_range=(bounds[r], bounds[r + 1]))
        parts.append((o, l.transpose(0, 2, 1)))
    o, l = oracle.attention(q, kc, vc, kt, vt, mask, part="tree")
    parts.append((o, l.transpose(0, 2, 1)))
    mo, ml = oracle.merge(parts)
    np.testing.assert_allclose(mo, full[0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ml.transpose(0, 2, 1), full[1], rtol=1e-12, atol=1e-12)


def test_merge_sentinel_identity_and_equal_parts():
    """The sentinel (0, -inf) is the merge identity; two parts with equal O keep O and add
    ln 2 to equal LSEs; two sentinels stay a sentinel (no NaN)."""
    rng = np.random.default_rng(0)
    o = rng.standard_normal((5, 8))
    l = rng.standard_normal(5) * 50
    mo, ml = oracle.merge([(o, l), (np.zeros_like(o), np.full(5, -np.inf))])
    np.testing.assert_array_equal(mo, o)
    np.testing.assert_array_equal(ml, l)
    mo, ml = oracle.merge([(o, l), (o, l)])
    np.testing.assert_allclose(mo, o, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(ml, l + math.log(2), rtol=1e-15, atol=1e-13)
    mo, ml = oracle.merge([(np.zeros_like(o), np.full(5, -np.inf))] * 2)
    assert np.all(mo == 0) and np.all(np.isneginf(ml))


def test_shift_invariance_and_scale_use():
    """I6: appending a constant column adds c to every logit of the row: O unchanged, LSE + c."""
    B, T, H, Hkv, d, N = 1, 3, 2, 1, 16, 20
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 50)
    mask = oracle.tree_mask(tree_parents("chain", T))[None]
    s, c = 0.25, 7.5
    o1, l1 = oracle.attention(q, kc, vc, kt, vt, mask, scale=s)
    ext = lambda x, val: torch.cat([x, torch.full(x.shape[:-1] + (1,), val)], -1)
    o2, l2 = oracle.attention(ext(q, c / s), ext(kc, 1.0), ext(vc, 0.0), ext(kt, 1.0), ext(vt, 0.0),
                              mask, scale=s)
    np.testing.assert_allclose(o2[..., :d], o1, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(l2, l1 + c, rtol=1e-12, atol=1e-12)


def test_key_permutation_invariance():
    """I7: permuting cache keys (with their values) changes nothing."""
    B, T, H, Hkv, d, N = 1, 4, 2, 2, 16, 31
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 60)
    mask = oracle.tree_mask(tree_parents("star", T))[None]
    perm = torch.randperm(N, generator=named_generator(0, "perm"))
    o1, l1 = oracle.attention(q, kc, vc, kt, vt, mask)
    o2, l2 = oracle.attention(q, kc[:, perm], vc[:, perm], kt, vt, mask)
    np.testing.assert_allclose(o2, o1, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(l2, l1, rtol=1e-13, atol=1e-13)


def test_naive_sum_exp_matches_for_bounded_logits():
    """I8: with |z| <= 80 the literal (unshifted) sum of exp equals the oracle within 1e-12,
    and logits in [-80, 80] never produce NaN/Inf."""
    B, T, H, Hkv, d, N = 1, 2, 1, 1, 4, 64
    q, kc, vc, kt, vt = oracle_inputs(B, T, H, Hkv, d, N, 70, q_scale=10.0)
    mask = np.ones((1, T, T), np.uint8)
    o, l = oracle.attention(q, kc, vc, kt, vt, mask, scale=1.0)
    assert np.all(np.isfinite(o)) and np.all(np.isfinite(l))
    K = torch.cat([kc[0, :, 0], kt[0, :, 0]]).double().numpy()
    V = torch.cat([vc[0, :, 0], vt[0, :, 0]]).double().numpy()
    for t in range(T):
        z = K @ q[0, t, 0].double().numpy()
        assert np.abs(z).max() <= 80
        e = np.exp(z)
        np.testing.assert_allclose(o[0, t, 0], (e @ V) / e.sum(), rtol=1e-12, atol=1e-12)
        assert abs(l[0, 0, t] - math.log(e.sum())) < 1e-12


def test_seqlens_exclude_garbage_tail():
    """Z13: columns j >= cache_seqlens[b] are excluded even when they hold NaN."""
    w = make_workload(2, 5, 4, 2, 32, 40, "fp32", dist="V1", seed=3,
                      seqlens=torch.tensor([40, 17], dtype=torch.int32), garbage_tail=True)
    mask = np.stack([oracle.tree_mask(w.parents[b]) for b in range(2)])
    o, l = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    assert np.all(np.isfinite(o)) and np.all(np.isfinite(l))
    o2, l2 = oracle.attention(w.q[1:], w.k_cache[1:, :17], w.v_cache[1:, :17], w.k_tree[1:], w.v_tree[1:],
                              mask[1:])
    np.testing.assert_array_equal(o[1:], o2)


def test_rows_subset_matches_full():
    w = make_workload(2, 6, 4, 2, 32, 70, "bf16", dist="V2", seed=4, tree="heap_binary")
    mask = np.stack([oracle.tree_mask(w.parents[b]) for b in range(2)])
    o, l = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    rows = [(1, 5, 3), (0, 0, 0), (1, 2, 1)]
    ro, rl = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, rows=rows)
    for i, (b, t, h) in enumerate(rows):
        np.testing.assert_array_equal(ro[i], o[b, t, h])
        assert rl[i] == l[b, h, t]
