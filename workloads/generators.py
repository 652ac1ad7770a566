"""Seeded generators for Hybrid-Tree-Attention workloads (no method arithmetic here).

Shapes follow BASELINE.json `configs`; value distributions and tree shapes follow the
recipe in DESIGN.md ("Input recipe"), which restates SURVEY.md §8(d):

* V0 "iid"          Q, K, V ~ N(0, 1).
* V1 "sink+local"   Q = 1.5 z + 8 u; planted prefix keys K = z + 16 u (the first four
                    positions -- the attention sinks of PAPER.md:169 footnote --, a seeded
                    1 % of positions and the last 64 valid positions); other keys K = z;
                    tree keys K_tree = z + 22 u; V, V_tree ~ N(0, 1).
* V2 "extreme"      Q = 3 z + 40 u; planted K = z + 24 u; K_tree = z + 24 u (logits ~85,
                    beyond fp32 exp overflow: exercises the max-shifted merge).

z is fresh N(0, I_d) per row, u is a seeded unit vector per (b, kv-head).

Trees are parent arrays with parents[i] < i (-1 = child of the committed context):
heap-binary (the toy "branching 2, depth 3"), chain, star, forest-of-roots, random
recursive, and `beam_tree` that mimics the dynamic beam search of PAPER.md:890
(widths [4,16,16,16,16], halted nodes kept, not removed).

Every tensor is drawn on the CPU from a torch.Generator seeded by (BASE_SEED, seed, name)
so the oracle and the GPU path see bit-identical inputs.
"""
from __future__ import annotations

import dataclasses
import zlib
from typing import Dict, Optional

import torch

BASE_SEED = 20250224

# BASELINE.json "configs", in order.  `N` is the prefix length (cache capacity N_max).
CONFIGS: Dict[str, dict] = {
    "toy": dict(B=1, T=8, H=1, H_kv=1, d=64, N=256, dtype="fp32", tree="heap_binary",
                desc="toy: 1 head, d=64, prefix N=256, 8-token tree (branching 2, depth 3), fp32"),
    "longchat7b_16k": dict(B=1, T=64, H=32, H_kv=32, d=128, N=16384, dtype="bf16", tree="beam",
                           desc="LongChat-7B-like: 32 MHA heads d=128, prefix 16k, 64-token tree, bf16"),
    "llama8b_64k": dict(B=1, T=64, H=32, H_kv=8, d=128, N=65536, dtype="bf16", tree="beam",
                        desc="Llama-3.1-8B-like GQA 32q/8kv d=128, prefix 64k, 64-token tree, bf16"),
    "qwq32b_32k_b4": dict(B=4, T=64, H=40, H_kv=8, d=128, N=32768, dtype="bf16", tree="beam",
                          desc="QwQ-32B-like GQA 40q/8kv d=128, prefix 32k, 64-token tree, batch 4"),
    "llama8b_128k_t128": dict(B=1, T=128, H=32, H_kv=8, d=128, N=131072, dtype="bf16", tree="beam",
                              desc="Llama-3.1-8B-like GQA, prefix 128k, 128-token tree"),
}


def named_generator(seed: int, name: str) -> torch.Generator:
    """A CPU generator for the named stream `name` of run `seed` (stable across processes)."""
    h = zlib.crc32(f"{BASE_SEED}:{seed}:{name}".encode())
    g = torch.Generator(device="cpu")
    g.manual_seed(h)
    return g


# --------------------------------------------------------------------------- trees

def tree_parents(kind: str, T: int, seed: int = 0) -> torch.Tensor:
    """Parent array int32[T] of the named shape."""
    if T <= 0:
        return torch.zeros(0, dtype=torch.int32)
    if kind == "heap_binary":
        p = [-1] + [(i - 1) // 2 for i in range(1, T)]
    elif kind == "chain":
        p = [i - 1 for i in range(T)]
    elif kind == "star":
        p = [-1] + [0] * (T - 1)
    elif kind == "roots":
        p = [-1] * T
    elif kind == "random":
        g = named_generator(seed, f"tree:random:{T}")
        p = [-1] + [int(torch.randint(0, i, (1,), generator=g)) for i in range(1, T)]
    elif kind == "random_forest":
        g = named_generator(seed, f"tree:random_forest:{T}")
        p = [int(torch.randint(-1, i, (1,), generator=g)) for i in range(T)]
    elif kind == "beam":
        return beam_tree(T, seed=seed)
    else:
        raise ValueError(f"unknown tree kind {kind!r}")
    return torch.tensor(p, dtype=torch.int32)


def beam_tree(T: int, widths=(4, 16, 16, 16, 16), seed: int = 0) -> torch.Tensor:
    """Tree shaped like LongSpec's dynamic beam search.

    Level 0 is the root (the pending token).  Level l gets widths[l-1] active nodes, each
    with a parent drawn uniformly from level l-1's active nodes.  While fewer than T nodes
    exist, halted leaves are added under uniformly drawn active nodes ("halt the
    computation of descendant nodes ... without removing them entirely").  Nodes are then
    stable-sorted by (depth, creation order) and truncated to T (a BFS order, so
    parents[i] < i holds).
    """
    g = named_generator(seed, f"tree:beam:{T}")
    nodes = [(0, -1)]  # (depth, parent creation id)
    levels = [[0]]
    for lvl, w in enumerate(widths, start=1):
        prev = levels[-1]
        cur = []
        for _ in range(w):
            par = prev[int(torch.randint(0, len(prev), (1,), generator=g))]
            nodes.append((lvl, par))
            cur.append(len(nodes) - 1)
        levels.append(cur)
    active = [i for lv in levels for i in lv]
    while len(nodes) < T:
        par = active[int(torch.randint(0, len(active), (1,), generator=g))]
        nodes.append((nodes[par][0] + 1, par))
    order = sorted(range(len(nodes)), key=lambda i: (nodes[i][0], i))[:T]
    new_id = {old: new for new, old in enumerate(order)}
    parents = [-1 if nodes[old][1] < 0 else new_id[nodes[old][1]] for old in order]
    return torch.tensor(parents, dtype=torch.int32)


def random_mask(B: int, T: int, density: float, seed: int, name: str = "mask") -> torch.Tensor:
    """An arbitrary 0/1 mask uint8[B,T,T] (not necessarily a tree); some rows may be empty."""
    g = named_generator(seed, f"{name}:{B}:{T}:{density}")
    return (torch.rand(B, T, T, generator=g) < density).to(torch.uint8)


def accept_tokens(parents: torch.Tensor, seed: int, vocab: int = 8, p_match: float = 0.7,
                  distinct_siblings: bool = True):
    """Synthetic (draft_tokens, target_argmax, context_argmax) for the accepted-path step.

    target_argmax[u] is the target's greedy token after node u.  Each child of u draws its
    draft token equal to target_argmax[u] with probability p_match (siblings distinct when
    `distinct_siblings`, as beam search proposes distinct tokens per parent).
    """
    T = parents.numel()
    g = named_generator(seed, f"accept:{T}:{vocab}:{p_match}:{distinct_siblings}")
    tgt = torch.randint(0, vocab, (T,), generator=g, dtype=torch.int64)
    ctx = int(torch.randint(0, vocab, (1,), generator=g))
    draft = torch.zeros(T, dtype=torch.int64)
    used: Dict[int, set] = {}
    for i in range(T):
        par = int(parents[i])
        want = ctx if par < 0 else int(tgt[par])
        seen = used.setdefault(par, set())
        if float(torch.rand(1, generator=g)) < p_match and (not distinct_siblings or want not in seen):
            tok = want
        else:
            tok = int(torch.randint(0, vocab, (1,), generator=g))
            if distinct_siblings:
                tries = 0
                while tok in seen and tries < 4 * vocab:
                    tok = int(torch.randint(0, vocab, (1,), generator=g))
                    tries += 1
                if tok in seen:  # vocabulary exhausted: use a fresh id outside it
                    tok = vocab + i
        seen.add(tok)
        draft[i] = tok
    return draft.to(torch.int32), tgt.to(torch.int32), ctx


# --------------------------------------------------------------------------- tensors

@dataclasses.dataclass
class Workload:
    """One synthetic verification-attention input (host tensors, exact bf16/fp32 values)."""
    B: int
    T: int
    H: int
    H_kv: int
    d: int
    N: int
    dtype: str
    dist: str
    seed: int
    q: torch.Tensor          # [B, T, H, d]
    k_cache: torch.Tensor    # [B, N, H_kv, d]
    v_cache: torch.Tensor    # [B, N, H_kv, d]
    k_tree: torch.Tensor     # [B, T, H_kv, d]
    v_tree: torch.Tensor     # [B, T, H_kv, d]
    parents: torch.Tensor    # int32 [B, T]
    seqlens: torch.Tensor    # int32 [B]
    scale: float

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32


def _unit(gen: torch.Generator, n: int, d: int) -> torch.Tensor:
    u = torch.randn(n, d, generator=gen)
    return u / u.norm(dim=-1, keepdim=True)


def make_workload(B: int, T: int, H: int, H_kv: int, d: int, N: int, dtype: str = "bf16",
                  dist: str = "V1", seed: int = 0, tree: str = "beam",
                  seqlens: Optional[torch.Tensor] = None, garbage_tail: bool = False) -> Workload:
    """Draw a workload.  `garbage_tail` fills cache rows >= seqlens[b] with NaN (Z13 test)."""
    assert H % H_kv == 0
    G = H // H_kv
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tag = f"{B}x{T}x{H}x{H_kv}x{d}x{N}:{dist}"
    if seqlens is None:
        seqlens = torch.full((B,), N, dtype=torch.int32)
    seqlens = seqlens.to(torch.int32)

    def randn(name, *shape):
        return torch.randn(*shape, generator=named_generator(seed, f"{tag}:{name}"))

    if dist == "V0":
        q = randn("q", B, T, H, d)
        kc = randn("kc", B, N, H_kv, d)
        kt = randn("kt", B, T, H_kv, d)
    elif dist in ("V1", "V2"):
        aq, ak, at = (1.5, 16.0, 22.0) if dist == "V1" else (3.0, 24.0, 24.0)
        bq = 8.0 if dist == "V1" else 40.0
        u = _unit(named_generator(seed, f"{tag}:u"), B * H_kv, d).view(B, H_kv, d)
        uq = u.repeat_interleave(G, dim=1)  # query head h uses u of its kv head h // G
        q = aq * randn("q", B, T, H, d) + bq * uq[:, None, :, :]
        kc = randn("kc", B, N, H_kv, d)
        gp = named_generator(seed, f"{tag}:planted")
        planted = torch.rand(B, N, generator=gp) < 0.01
        planted[:, :4] = True
        for b in range(B):
            n = int(seqlens[b])
            planted[b, max(0, n - 64):n] = True
        kc = kc + ak * planted[:, :, None, None].float() * u[:, None, :, :]
        kt = randn("kt", B, T, H_kv, d) + at * u[:, None, :, :]
    else:
        raise ValueError(dist)
    vc = randn("vc", B, N, H_kv, d)
    vt = randn("vt", B, T, H_kv, d)

    if garbage_tail:
        for b in range(B):
            n = int(seqlens[b])
            kc[b, n:] = float("nan")
            vc[b, n:] = float("nan")

    parents = torch.stack([tree_parents(tree, T, seed=seed * 1000 + b) for b in range(B)]) \
        if T > 0 else torch.zeros(B, 0, dtype=torch.int32)
    scale = float(torch.tensor(1.0 / d ** 0.5, dtype=torch.float32))
    return Workload(B, T, H, H_kv, d, N, dtype, dist, seed,
                    q.to(tdt), kc.to(tdt), vc.to(tdt), kt.to(tdt), vt.to(tdt),
                    parents.to(torch.int32), seqlens, scale)


def config_workload(name: str, dist: str = "V1", seed: int = 0, **over) -> Workload:
    c = dict(CONFIGS[name])
    c.pop("desc")
    c.update(over)
    return make_workload(c["B"], c["T"], c["H"], c["H_kv"], c["d"], c["N"], c["dtype"],
                         dist=dist, seed=seed, tree=c["tree"])


def fp8_cache(x: torch.Tensor):
    """An E4M3 copy of a cache tensor [B, N, H_kv, d] for the FP8-cache row:
    per KV head a power-of-two scale (2^ceil(log2(amax / 448)), so that scale * E4M3 is exact in
    float32) and the E4M3 bytes of x / scale (torch's round-to-nearest conversion).  Returns
    (bytes uint8 [B, N, H_kv, d], scale float32 [H_kv]).  Input generation only: the E4M3 values
    are the inputs both the oracle and the GPU path decode."""
    xf = x.float()
    finite = torch.where(torch.isfinite(xf), xf.abs(), torch.zeros_like(xf))
    amax = finite.amax(dim=(0, 1, 3)).clamp_min(1e-30)
    scale = torch.exp2(torch.ceil(torch.log2(amax / 448.0)))
    q8 = (xf / scale[None, None, :, None]).to(torch.float8_e4m3fn)
    return q8.view(torch.uint8), scale.to(torch.float32)
