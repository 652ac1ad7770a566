"""Diagnostics: per-row prefix errors vs the oracle for a few shapes and forced split counts (used
to localise the polynomial-exp overflow; run against variant libraries via tools/lib_variants.sh)."""
import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload
dev = torch.device("cuda:0")
for case in [(2, 33, 8, 8, 64, 2049, "V2"), (3, 1, 32, 8, 64, 1500, "V2"), (2, 33, 8, 8, 64, 2049, "V1"), (2, 33, 8, 8, 128, 2049, "V2")]:
    B, T, H, Hkv, d, N, dist = case
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist=dist, seed=7, tree="random")
    mask = np.stack([oracle.tree_mask(w.parents[b]) for b in range(B)])
    oc_ref, lc_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, part="cache")
    q, kc, vc = w.q.to(dev), w.k_cache.to(dev), w.v_cache.to(dev)
    for S in (0, 1, 2, 3, 5, 8):
        oc, lc = hta.hta_prefix_attn(q, kc, vc, num_splits=S)
        torch.cuda.synchronize()
        err = (oc.cpu().double().numpy() - oc_ref).__abs__().max(axis=-1)  # [B,T,H]
        lerr = np.abs(lc.cpu().double().numpy() - lc_ref)
        bad = np.argwhere(err > 0.05)
        print(case, "S", S, "max err", err.max(), "lse err", lerr.max(), "bad rows", len(bad), bad[:6].tolist())
