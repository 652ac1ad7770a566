"""Pins of oracle.commit_kv (SPEC commit_kv S:212-220), independent of it.

* prefill equivalence (and the losslessness of PAPER.md:190): after committing the
  accepted path, the attention of path node i over the committed cache rows [0, n + i + 1)
  equals its tree attention (prefix n + its visible ancestors) from the verification step.
  Attention is permutation-invariant over keys, but the visible row SETS of the intermediate
  nodes depend on the order, so a wrong order or a wrong row fails here;
* a hand-worked example, rows outside the appended range untouched, empty path, saturation at
  N_max (reading Z18).
"""
import numpy as np
import pytest
import torch

import oracle
from workloads import make_workload


def test_commit_hand_worked_example():
    # cache rows hold their own index, tree rows hold 100 + node: n = 2, path [0, 2, 3]
    B, N, Hkv, d, T = 1, 7, 1, 2, 4
    kc = np.arange(N, dtype=np.float64).reshape(1, N, 1, 1).repeat(d, axis=3)
    kt = (100 + np.arange(T, dtype=np.float64)).reshape(1, T, 1, 1).repeat(d, axis=3)
    k2, v2, n2 = oracle.commit_kv(kc, -kc, [2], kt, -kt, [[0, 2, 3, 1]], [3])
    assert k2[0, :, 0, 0].tolist() == [0, 1, 100, 102, 103, 5, 6]
    assert v2[0, :, 0, 0].tolist() == [0, -1, -100, -102, -103, -5, -6]
    assert n2.tolist() == [5]


def test_commit_empty_path_and_saturation():
    B, N, Hkv, d, T = 2, 5, 2, 4, 3
    rng = np.random.default_rng(0)
    kc, vc = rng.normal(size=(2, B, N, Hkv, d))
    kt, vt = rng.normal(size=(2, B, T, Hkv, d))
    k2, v2, n2 = oracle.commit_kv(kc, vc, [1, 3], kt, vt, [[0, 1, 2], [0, 1, 2]], [0, 3])
    np.testing.assert_array_equal(k2[0], kc[0])           # empty acceptance: unchanged
    np.testing.assert_array_equal(k2[1, :3], kc[1, :3])   # untouched prefix
    np.testing.assert_array_equal(k2[1, 3], kt[1, 0])
    np.testing.assert_array_equal(k2[1, 4], kt[1, 1])     # node 2 would land at 5 = N_max: dropped
    assert n2.tolist() == [1, 5]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_commit_prefill_equivalence(seed):
    B, T, H, Hkv, d, N = 2, 24, 4, 2, 32, 300
    w = make_workload(B, T, H, Hkv, d, N, "fp32", dist="V1", seed=seed, tree="beam")
    rng = np.random.default_rng(seed)
    n0 = np.array([200, 137])
    masks = np.stack([oracle.tree_mask(w.parents[b]) for b in range(B)])
    o_tree, _ = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, masks, seqlens=n0)
    paths, lens = [], []
    for b in range(B):
        par = w.parents[b].tolist()
        # an accepted path: a random deepest root-to-leaf chain
        leaf = int(rng.integers(T // 2, T))
        chain = [leaf]
        while par[chain[-1]] >= 0:
            chain.append(par[chain[-1]])
        path = chain[::-1]
        paths.append(path + [0] * (T - len(path)))
        lens.append(len(path))
        assert len(path) >= 2
    k2, v2, n2 = oracle.commit_kv(w.k_cache.numpy(), w.v_cache.numpy(), n0, w.k_tree.numpy(), w.v_tree.numpy(),
                                  paths, lens)
    assert n2.tolist() == [int(n0[b] + lens[b]) for b in range(B)]
    no_tree = np.zeros((1, 1, 1), np.uint8)
    for b in range(B):
        for i, v in enumerate(paths[b][:lens[b]]):
            q1 = w.q[b:b + 1, v:v + 1]
            o_c, _ = oracle.attention(q1, torch.from_numpy(k2[b:b + 1]), torch.from_numpy(v2[b:b + 1]),
                                      w.k_tree[b:b + 1, :1], w.v_tree[b:b + 1, :1], no_tree,
                                      seqlens=np.array([n0[b] + i + 1]), part="cache")
            np.testing.assert_allclose(o_c[0, 0], o_tree[b, v], rtol=0, atol=1e-12)
        # rows past the appended range are untouched
        e = int(n0[b] + lens[b])
        np.testing.assert_array_equal(k2[b, e:], w.k_cache.numpy()[b, e:])
        np.testing.assert_array_equal(k2[b, :n0[b]], w.k_cache.numpy()[b, :n0[b]])
