"""Tree-mask and accepted-path oracles -- TEST INFRASTRUCTURE ONLY.

tree_mask      PAPER.md:191 ("attention masks derived from prefix trees ... disabling wrong
               combinations between speculation tokens") and PAPER.md:225 (mask applied per
               block).  Reading Z4: allow[i][j] = 1 iff j == i or j is an ancestor of i.
               Built by walking each node's parent chain into a Python set (recursively),
               then written as a dense 0/1 matrix -- independent of the bit-parallel
               builder in the product.
accept_greedy  PAPER.md:190 (the target verifies the tree "without altering the final
               results") and the greedy acceptance of PAPER.md:239/449 (T=0, tau = mean
               accepted tokens per target forward).  Reading Z12: the accepted path is the
               LONGEST root-anchored path whose every node's draft token equals the target
               argmax at its parent; ties -> lexicographically smallest node-index sequence;
               bonus = target argmax at the path's last node.  Computed by brute force over
               every node's root path.
commit_kv      PAPER.md:172 ("the large model only updates its KV cache upon verification
               completion") and SPEC commit_kv: the cache is extended by exactly
               the accepted nodes' K/V rows in path order; rejected rows are discarded.
               Plain row-by-row copy.  Rows that would land at or beyond N_max are dropped
               (the committed length saturates at N_max: reading Z18).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def _as_list(x) -> List[int]:
    if hasattr(x, "tolist"):
        return [int(v) for v in x.tolist()]
    return [int(v) for v in x]


def _ancestors(parents: List[int], i: int) -> set:
    """Recursive ancestor set of node i (its parent, and the parent's ancestors)."""
    p = parents[i]
    if p < 0:
        return set()
    return {p} | _ancestors(parents, p)


def validate_parents(parents: Sequence[int]) -> None:
    """Reading Z6: nodes are in topological order, parents[i] in [-1, i)."""
    for i, p in enumerate(parents):
        if not (-1 <= p < i):
            raise ValueError(f"parents[{i}] = {p} violates -1 <= parents[i] < i")


def tree_mask(parents) -> np.ndarray:
    """Dense uint8 [T, T] ancestor mask (1 = node j visible to node i)."""
    par = _as_list(parents)
    validate_parents(par)
    T = len(par)
    m = np.zeros((T, T), np.uint8)
    for i in range(T):
        for j in _ancestors(par, i) | {i}:
            m[i, j] = 1
    return m


def accept_greedy(parents, draft_tokens, target_argmax, root: int = 0,
                  context_argmax: int = -1) -> Tuple[List[int], int]:
    """(path, bonus) of the longest accepted path.

    root >= 0: the walk starts at node `root` (path[0] == root; root is always accepted).
    root == -1: forest mode; nodes with parents == -1 hang under the committed context and
    are matched against `context_argmax`; the path may be empty (bonus = context_argmax).
    """
    par = _as_list(parents)
    validate_parents(par)
    draft = _as_list(draft_tokens)
    tgt = _as_list(target_argmax)
    T = len(par)
    if root >= 0 and not (0 <= root < T):
        raise ValueError("root out of range")
    candidates = []
    for v in range(T):
        # the chain v -> ... -> top (a node with parent -1)
        chain = [v]
        while par[chain[-1]] != -1:
            chain.append(par[chain[-1]])
        chain = chain[::-1]
        if root >= 0:
            if root not in chain:
                continue
            path = chain[chain.index(root):]
            ok = all(draft[u] == tgt[par[u]] for u in path[1:])
        else:
            path = chain
            ok = draft[path[0]] == context_argmax and all(draft[u] == tgt[par[u]] for u in path[1:])
        if ok:
            candidates.append(path)
    if not candidates:
        return [], int(context_argmax)
    best_len = max(len(p) for p in candidates)
    best = min(p for p in candidates if len(p) == best_len)  # lexicographic on index lists
    return best, int(tgt[best[-1]])


def commit_kv(k_cache, v_cache, seqlens, k_tree, v_tree, paths, path_lens):
    """(k_cache', v_cache', seqlens') after appending, for every batch b, the tree K/V rows of
    nodes paths[b][0 .. path_lens[b]) at cache positions seqlens[b], seqlens[b] + 1, ...

    k_cache/v_cache [B, N, H_kv, d]; k_tree/v_tree [B, T, H_kv, d]; seqlens [B]; paths [B][>= len];
    path_lens [B].  Inputs are not modified (numpy copies are returned).
    """
    kc = np.array(k_cache, copy=True)
    vc = np.array(v_cache, copy=True)
    kt = np.asarray(k_tree)
    vt = np.asarray(v_tree)
    B, N = kc.shape[0], kc.shape[1]
    T = kt.shape[1]
    out_len = []
    for b in range(B):
        n = int(seqlens[b])
        L = int(path_lens[b])
        path = [int(x) for x in paths[b][:L]]
        for i, node in enumerate(path):
            if not 0 <= node < T:
                raise ValueError(f"path node {node} outside [0, {T})")
            if n + i >= N:
                break
            kc[b, n + i] = kt[b, node]
            vc[b, n + i] = vt[b, node]
        out_len.append(min(n + L, N))
    return kc, vc, np.asarray(out_len, np.int64)
