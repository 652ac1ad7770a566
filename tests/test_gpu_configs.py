"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(default split plan): every row of the headline config (Llama-8B-64k, 2048 rows), >= 1024 rows of
QwQ-32k x 4 and of Llama-8B-128k/T=128, and rows sampled across every KV head, tree depth and batch
for the other configs / distributions; the oracle computes exactly those rows (fp64, explicit
mask, all host cores)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import CONFIGS
from workloads.generators import config_workload, named_generator

from gpu_util import compare, oracle_masks, to_dev

pytestmark = pytest.mark.gpu


def sample_rows(B, T, H, n, seed):
    if n >= B * T * H:  # every row
        return [(b, t, h) for b in range(B) for t in range(T) for h in range(H)]
    g = named_generator(seed, "rows")
    rows = {(0, 0, 0), (B - 1, T - 1, H - 1)}
    while len(rows) < n:
        rows.add((int(torch.randint(0, B, (1,), generator=g)), int(torch.randint(0, T, (1,), generator=g)),
                  int(torch.randint(0, H, (1,), generator=g))))
    return sorted(rows)


@pytest.mark.parametrize("name,dist", [(n, "V1") for n in CONFIGS] +
                         [("llama8b_64k", "V2"), ("qwq32b_32k_b4", "V2"), ("longchat7b_16k", "V0"),
                          ("llama8b_128k_t128", "V2")])
def test_config_full_size_sampled(cuda_device, name, dist):
    w = config_workload(name, dist=dist, seed=0)
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                           cache_seqlens=x["sl"])
    torch.cuda.synchronize()
    n_all = w.B * w.T * w.H
    want = {"llama8b_64k": n_all, "qwq32b_32k_b4": 1024, "llama8b_128k_t128": 1024}.get(name, 64) if dist == "V1" else 64
    rows = sample_rows(w.B, w.T, w.H, min(n_all, want) if w.N > 1000 else n_all, seed=1)
    ro, rl = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens, rows=rows)
    idx = torch.tensor(rows)
    og = o[idx[:, 0], idx[:, 1], idx[:, 2]]
    lg = l[idx[:, 0], idx[:, 2], idx[:, 1]]
    stats = compare(og, lg, ro, rl, w.dtype, name)
    print(name, dist, stats)
    # properties that hold at any size, on every row: finite, no NaN, LSE >= the prefix LSE
    assert torch.isfinite(o.float()).all() and torch.isfinite(l).all()


@pytest.mark.parametrize("T", [16, 4])
def test_draft_cross_attention_full_size(cuda_device, T):
    """the draft model's cross-attention over the target's KV cache is the
    same unmasked prefix contraction with a small M (queries = the beam frontier, <= 16 tokens x
    G): hta_prefix_attn at the Llama-8B-64k cache size, sampled rows vs the oracle's cache part."""
    w = config_workload("llama8b_64k", dist="V1", seed=3)
    q = w.q[:, :T].contiguous()
    x = to_dev(w, cuda_device)
    o, l = hta.hta_prefix_attn(q.to(cuda_device), x["kc"], x["vc"])
    torch.cuda.synchronize()
    rows = sample_rows(w.B, T, w.H, 48, seed=2)
    mask = np.zeros((w.B, T, T), np.uint8)
    ro, rl = oracle.attention(q, w.k_cache, w.v_cache, w.k_tree[:, :T], w.v_tree[:, :T], mask, part="cache",
                              rows=rows)
    idx = torch.tensor(rows)
    compare(o[idx[:, 0], idx[:, 1], idx[:, 2]], l[idx[:, 0], idx[:, 2], idx[:, 1]], ro, rl, "bf16", f"xattn T={T}")


@pytest.mark.parametrize("name", ["qwq32b_32k_b4", "longchat7b_16k", "llama8b_64k"])
def test_fp8kv_full_size_sampled(cuda_device, name):
    """SURVEY.md §8(f) f4 at full size: hta_forward_fp8kv over an E4M3 copy of the config's cache
    (per-KV-head power-of-two scales), sampled rows against the oracle over the decoded cache.
    QwQ runs the split-P PV variant (single CTAs of more than 64 rows), LongChat the E4M3 S path
    with V widened (64-row units), Llama the CTA-pair path with K and V widened."""
    from workloads import fp8_cache
    w = config_workload(name, dist="V1", seed=0)
    mask = oracle_masks(w)
    k8, ks = fp8_cache(w.k_cache)
    v8, vs = fp8_cache(w.v_cache)
    dev = cuda_device
    o, l = hta.hta_forward_fp8kv(w.q.to(dev), k8.to(dev), v8.to(dev), ks.to(dev), vs.to(dev), w.k_tree.to(dev),
                                 w.v_tree.to(dev), torch.from_numpy(mask).to(dev), cache_seqlens=w.seqlens.to(dev))
    torch.cuda.synchronize()
    rows = sample_rows(w.B, w.T, w.H, 256, seed=2)
    ro, rl = oracle.attention_fp8kv(w.q, k8, v8, ks, vs, w.k_tree, w.v_tree, mask, seqlens=w.seqlens, rows=rows)
    idx = torch.tensor(rows)
    compare(o[idx[:, 0], idx[:, 1], idx[:, 2]], l[idx[:, 0], idx[:, 2], idx[:, 1]], ro, rl, "bf16", f"fp8 {name}")
    assert torch.isfinite(o.float()).all() and torch.isfinite(l).all()
