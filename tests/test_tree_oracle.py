"""Pins of the tree-mask and accepted-path oracles (CPU only)."""
import itertools
import os

import numpy as np
import pytest
import torch

import oracle
from workloads import accept_tokens, beam_tree, tree_parents
from workloads.generators import named_generator

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_golden_mask():
    rows, parents = [], None
    for line in open(os.path.join(GOLDEN, "toy_tree_mask.txt")):
        line = line.strip()
        if line.startswith("# parents:"):
            parents = [int(x) for x in line.split(":")[1].split()]
        elif line and not line.startswith("#"):
            rows.append([int(c) for c in line])
    return parents, np.array(rows, np.uint8)


def load_accept_examples():
    out = []
    for line in open(os.path.join(GOLDEN, "accept_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = [x.strip() for x in line.split(";")]
        ints = lambda s: [int(x) for x in s.split()] if s else []
        out.append(dict(name=f[0], root=int(f[1]), ctx=int(f[2]), draft=ints(f[3]), tgt=ints(f[4]),
                        path=ints(f[5]), bonus=int(f[6])))
    return out


def greedy_walk(parents, draft, tgt, root=0, ctx=-1):
    """Textbook greedy walk: step to the lowest-index child whose draft token
    equals the target argmax at the current node; bonus = target argmax where it stops."""
    par = [int(p) for p in parents]
    T = len(par)
    if root >= 0:
        path, want, cur = [root], int(tgt[root]), root
    else:
        path, want, cur = [], ctx, -1
    while True:
        nxt = [c for c in range(T) if par[c] == cur and int(draft[c]) == want]
        if not nxt:
            return path, want
        cur = nxt[0]
        path.append(cur)
        want = int(tgt[cur])


# ------------------------------------------------------------------------ masks

def test_toy_mask_golden():
    parents, rows = load_golden_mask()
    assert parents == tree_parents("heap_binary", 8).tolist()
    m = oracle.tree_mask(parents)
    np.testing.assert_array_equal(m, rows)
    assert int(m.sum()) == 21


@pytest.mark.parametrize("T", [1, 2, 7, 64])
def test_chain_star_roots(T):
    np.testing.assert_array_equal(oracle.tree_mask(tree_parents("chain", T)), np.tril(np.ones((T, T), np.uint8)))
    star = np.eye(T, dtype=np.uint8)
    star[:, 0] = 1
    np.testing.assert_array_equal(oracle.tree_mask(tree_parents("star", T)), star)
    np.testing.assert_array_equal(oracle.tree_mask(tree_parents("roots", T)), np.eye(T, dtype=np.uint8))


@pytest.mark.parametrize("kind", ["random", "random_forest", "beam"])
def test_mask_recurrence_and_depth(kind):
    """allow[i] = allow[parent(i)] + e_i (row recurrence, a different formula) and
    popcount(row i) = depth(i) + 1 on seeded random trees up to T = 256."""
    for seed in range(20):
        T = [5, 64, 128, 256][seed % 4]
        par = tree_parents(kind, T, seed=seed).tolist()
        m = oracle.tree_mask(par)
        depth = []
        for i in range(T):
            want = np.zeros(T, np.uint8) if par[i] < 0 else m[par[i]].copy()
            want[i] = 1
            np.testing.assert_array_equal(m[i], want)
            depth.append(0 if par[i] < 0 else depth[par[i]] + 1)
            assert int(m[i].sum()) == depth[i] + 1
        # reflexive, and allow[i][j] => j <= i (topological order)
        assert np.all(np.diag(m) == 1) and np.all(np.triu(m, 1) == 0)


def test_beam_tree_shape():
    """beam_tree follows PAPER.md:890: widths [4,16,16,16,16] (<= 69 active nodes), halted
    nodes kept, BFS order (parents[i] < i), depth <= 5 (+1 for halted leaves)."""
    for T in (64, 128):
        par = beam_tree(T).tolist()
        assert len(par) == T and par[0] == -1
        assert all(-1 <= p < i for i, p in enumerate(par))
        depth = []
        for i, p in enumerate(par):
            depth.append(0 if p < 0 else depth[p] + 1)
        assert max(depth) <= 6
        if T <= 69:   # truncation of the active tree only: exactly 4 depth-1 nodes
            assert sum(1 for x in depth if x == 1) == 4 and max(depth) <= 5
        else:         # 69 active nodes + halted leaves (halted leaves may hang under the root)
            assert sum(1 for x in depth if x == 1) >= 4


def test_invalid_parents_rejected():
    for bad in ([0], [-1, 1], [-1, 0, 5], [-2]):
        with pytest.raises(ValueError):
            oracle.tree_mask(bad)


# ------------------------------------------------------------------------ accepted path

@pytest.mark.parametrize("ex", load_accept_examples(), ids=lambda e: e["name"])
def test_accept_golden(ex):
    par = tree_parents("heap_binary", 8).tolist()
    path, bonus = oracle.accept_greedy(par, ex["draft"], ex["tgt"], root=ex["root"], context_argmax=ex["ctx"])
    assert path == ex["path"] and bonus == ex["bonus"]


def test_accept_equals_greedy_walk_with_distinct_siblings():
    """With distinct sibling tokens (beam search proposes distinct tokens per parent,
    PAPER.md:890) the longest accepted path is the textbook greedy walk."""
    for seed in range(300):
        T = [1, 3, 8, 17, 64][seed % 5]
        kind = ["random", "beam", "chain", "star", "heap_binary"][seed % 5]
        par = tree_parents(kind, T, seed=seed)
        draft, tgt, ctx = accept_tokens(par, seed, vocab=6, p_match=0.75)
        for root in (0, -1):
            want = greedy_walk(par.tolist(), draft.tolist(), tgt.tolist(), root, ctx)
            got = oracle.accept_greedy(par, draft, tgt, root=root, context_argmax=ctx)
            assert got == (want[0], want[1]), (seed, root)


def test_accept_losslessness_vs_vanilla_greedy():
    """PAPER.md:190 ("without altering the final results"): with a deterministic target
    f(prefix) -> next token, the emitted tokens (draft tokens on the accepted path + bonus)
    equal the first tokens of vanilla greedy decoding, and no longer accepted prefix exists."""
    def f(seq):
        h = 7
        for x in seq:
            h = (h * 31 + x + 3) % 1009
        return h % 5

    for seed in range(200):
        g = named_generator(seed, "lossless")
        T = 1 + seed % 24
        par = tree_parents("random_forest", T, seed=seed).tolist()
        draft = torch.randint(0, 5, (T,), generator=g).tolist()
        ctx_seq = torch.randint(0, 5, (4,), generator=g).tolist()

        def node_seq(v):
            chain = [v]
            while par[chain[-1]] >= 0:
                chain.append(par[chain[-1]])
            return [draft[u] for u in chain[::-1]]

        tgt = [f(ctx_seq + node_seq(v)) for v in range(T)]
        path, bonus = oracle.accept_greedy(par, draft, tgt, root=-1, context_argmax=f(ctx_seq))
        emitted = [draft[u] for u in path] + [bonus]
        vanilla = []
        for _ in range(len(emitted)):
            vanilla.append(f(ctx_seq + vanilla))
        assert emitted == vanilla
        # maximality: no node's full token sequence matches a longer vanilla prefix
        longer = [f(ctx_seq)]
        for _ in range(len(path) + 1):
            longer.append(f(ctx_seq + longer))
        for v in range(T):
            s = node_seq(v)
            if len(s) > len(path):
                assert s != longer[:len(s)]


def test_accept_duplicate_siblings_takes_longest():
    """Reading Z12: with duplicate sibling tokens the longest path wins even when the
    first matching child is a dead end; among equal lengths the smaller index path wins."""
    par = [-1, 0, 0, 2, 0, 4]          # children of 0: 1 (leaf), 2 -> 3, 4 -> 5
    draft = [9, 5, 5, 6, 5, 6]
    tgt = [5, 0, 6, 1, 6, 2]
    path, bonus = oracle.accept_greedy(par, draft, tgt, root=0)
    assert path == [0, 2, 3] and bonus == 1
    # greedy walk would stop at the dead end 1
    assert greedy_walk(par, draft, tgt)[0] == [0, 1]


def test_accept_brute_force_small_trees():
    """Exhaustive over all 24 parent arrays of T <= 4 and all token patterns over {0,1}:
    path is accepted (every step matches), has maximal length, and is lexicographically
    smallest among the maximal ones (checked by enumerating every node's root path)."""
    for T in range(1, 5):
        for par in itertools.product(*[range(-1, i) for i in range(T)]):
            for bits in range(1 << T):
                draft = [(bits >> i) & 1 for i in range(T)]
                tgt = [(bits >> ((i + 1) % T)) & 1 for i in range(T)]
                path, bonus = oracle.accept_greedy(list(par), draft, tgt, root=-1, context_argmax=1)
                ok = []
                for v in range(T):
                    ch = [v]
                    while par[ch[-1]] >= 0:
                        ch.append(par[ch[-1]])
                    ch = ch[::-1]
                    if draft[ch[0]] == 1 and all(draft[u] == tgt[par[u]] for u in ch[1:]):
                        ok.append(ch)
                if not ok:
                    assert path == [] and bonus == 1
                else:
                    L = max(map(len, ok))
                    assert path == sorted(c for c in ok if len(c) == L)[0]
                    assert bonus == tgt[path[-1]]
