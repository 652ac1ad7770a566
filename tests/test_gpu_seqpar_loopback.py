"""Sequence-parallel step (row a5 of SURVEY.md §8) at P = 2, 4, 8 on ONE GPU through libhta's
loopback communicator (hta_comm_create_loopback / hta_forward_seqpar_loopback): each virtual rank
runs the same per-rank code as hta_forward_seqpar -- the local split-KV prefix pass over its
contiguous KV shard combined into destination-major blocks, the all-to-all of head slices (here
device copies), the P-way merge with the tree pass at head offset r*H/P (PAPER.md:207-218 applied
P+1 ways, Appendix C), and the optional all-gather + reassembly.  Every rank's output
is compared element by element with the one-shot fp64 oracle over the whole prefix + tree.

Shards are padded to a common capacity with NaN rows past each shard's valid length (they must
never reach the softmax, reading Z13), and the valid length can end before the last shards,
which then hold no key at all (their partial is the sentinel, reading Z10)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload

from gpu_util import compare, oracle_masks

pytestmark = pytest.mark.gpu


def _shards(w, P, seqlen, dev):
    """Per-rank KV slices (common capacity, NaN padding) and valid lengths."""
    bounds = [hta.shard_bounds(w.N, P, r) for r in range(P)]
    cap = max(hi - lo for lo, hi in bounds)
    ks, vs, sls = [], [], []
    for lo, hi in bounds:
        k = torch.full((w.B, cap, w.H_kv, w.d), float("nan"), dtype=w.k_cache.dtype)
        v = torch.full_like(k, float("nan"))
        k[:, :hi - lo] = w.k_cache[:, lo:hi]
        v[:, :hi - lo] = w.v_cache[:, lo:hi]
        ks.append(k.to(dev))
        vs.append(v.to(dev))
        sls.append(torch.clamp(seqlen - lo, 0, hi - lo).to(torch.int32).to(dev))
    return ks, vs, sls


CASES = [
    # B, T, H, Hkv, d, N, dtype, tree, P
    (1, 64, 32, 8, 128, 3000, "bf16", "beam", 2),
    (1, 64, 32, 8, 128, 3000, "bf16", "beam", 4),
    (1, 64, 32, 8, 128, 3000, "bf16", "beam", 8),
    (2, 13, 8, 2, 128, 1000, "bf16", "random", 8),
    (1, 9, 8, 2, 64, 700, "bf16", "star", 4),
    (1, 128, 32, 8, 128, 4100, "bf16", "beam", 8),
    (1, 8, 4, 1, 64, 256, "fp32", "heap_binary", 2),
    (1, 8, 4, 1, 64, 256, "fp32", "heap_binary", 4),
]


@pytest.mark.parametrize("gather", [False, True])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"B{c[0]}T{c[1]}H{c[2]}/{c[3]}d{c[4]}N{c[5]}{c[6]}P{c[8]}")
def test_loopback_ranks_vs_oracle(cuda_device, case, gather):
    B, T, H, Hkv, d, N, dtype, tree, P = case
    w = make_workload(B, T, H, Hkv, d, N, dtype, dist="V1", seed=11, tree=tree)
    mask = oracle_masks(w)
    ks, vs, sls = _shards(w, P, w.seqlens, cuda_device)
    comm = hta.LoopbackComm(P)
    try:
        os_, ls = comm.forward(w.q.to(cuda_device), ks, vs, w.k_tree.to(cuda_device), w.v_tree.to(cuda_device),
                               torch.from_numpy(mask).to(cuda_device), seqlens_slices=sls, gather_output=gather)
        torch.cuda.synchronize()
    finally:
        comm.close()
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    Hp = H // P
    for r in range(P):
        if gather:
            compare(os_[r], ls[r], o_ref, l_ref, dtype, f"P={P} rank {r} gathered")
            if r > 0:  # every rank ends with the same reassembled output
                assert torch.equal(os_[r], os_[0]) and torch.equal(ls[r], ls[0])
        else:
            hs = slice(r * Hp, (r + 1) * Hp)
            compare(os_[r], ls[r], o_ref[:, :, hs], l_ref[:, hs], dtype, f"P={P} rank {r} heads {hs}")


@pytest.mark.parametrize("P", [2, 8])
def test_loopback_empty_shards(cuda_device, P):
    """The valid prefix ends inside the first shard: ranks >= 1 hold no valid key (sentinel
    partials that must not disturb the merge), and one batch entry has no prefix at all."""
    B, T, H, Hkv, d, N = 2, 16, 16, 4, 128, 2048
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist="V1", seed=3, tree="random")
    seqlens = torch.tensor([N // (2 * P), 0], dtype=torch.int32)
    mask = oracle_masks(w)
    ks, vs, sls = _shards(w, P, seqlens, cuda_device)
    comm = hta.LoopbackComm(P)
    try:
        os_, ls = comm.forward(w.q.to(cuda_device), ks, vs, w.k_tree.to(cuda_device), w.v_tree.to(cuda_device),
                               torch.from_numpy(mask).to(cuda_device), seqlens_slices=sls, gather_output=True)
        torch.cuda.synchronize()
    finally:
        comm.close()
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=seqlens)
    for r in range(P):
        compare(os_[r], ls[r], o_ref, l_ref, "bf16", f"P={P} rank {r} (empty shards)")


def test_loopback_p1_equals_forward(cuda_device):
    """P = 1 loopback = the one-GPU forward up to the extra combine step (same tolerance)."""
    w = make_workload(1, 64, 32, 8, 128, 2500, "bf16", dist="V1", seed=4, tree="beam")
    mask = torch.from_numpy(oracle_masks(w)).to(cuda_device)
    x = {k: getattr(w, k).to(cuda_device) for k in ("q", "k_cache", "v_cache", "k_tree", "v_tree")}
    comm = hta.LoopbackComm(1)
    try:
        os_, ls = comm.forward(x["q"], [x["k_cache"]], [x["v_cache"]], x["k_tree"], x["v_tree"], mask)
        o1, l1 = hta.hta_forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], mask)
        torch.cuda.synchronize()
        assert (os_[0].float() - o1.float()).abs().max().item() <= 2e-2
        assert (ls[0] - l1).abs().max().item() <= 1e-4
    finally:
        comm.close()


P2P_CASES = [
    # B, T, H, Hkv, d, N, dtype, tree, P
    (1, 64, 32, 8, 128, 3000, "bf16", "beam", 2),
    (1, 64, 32, 8, 128, 3000, "bf16", "beam", 8),
    (2, 13, 8, 2, 128, 1000, "bf16", "random", 4),
    (1, 128, 32, 8, 128, 4100, "bf16", "beam", 8),
    (1, 8, 4, 1, 64, 256, "fp32", "heap_binary", 2),
]


@pytest.mark.parametrize("case", P2P_CASES, ids=lambda c: f"B{c[0]}T{c[1]}H{c[2]}/{c[3]}d{c[4]}N{c[5]}{c[6]}P{c[8]}")
def test_loopback_peer_memory_exchange(cuda_device, case):
    """The peer-memory exchange (hta_comm_p2p_*): each virtual rank's split combine writes its
    head blocks straight into the other ranks' receive buffers, a signal kernel raises its flag
    in every rank's flag array, each final merge waits for all P flags.  Three consecutive steps
    on different inputs exercise both halves of the double-buffered receive buffers and the step
    counters; every step's every rank equals the copy-exchange loopback step bit for bit and the
    oracle within tolerance."""
    B, T, H, Hkv, d, N, dtype, tree, P = case
    p2p = hta.LoopbackComm(P)
    ref = hta.LoopbackComm(P)
    try:
        for step in range(3):
            w = make_workload(B, T, H, Hkv, d, N, dtype, dist="V1", seed=40 + step, tree=tree)
            mask = torch.from_numpy(oracle_masks(w)).to(cuda_device)
            ks, vs, sls = _shards(w, P, w.seqlens, cuda_device)
            shape = hta.make_shape(w.q.to(cuda_device), k_cache=ks[0], k_tree=w.k_tree.to(cuda_device))
            if step == 0:
                p2p.enable_p2p([shape])
            args = (w.q.to(cuda_device), ks, vs, w.k_tree.to(cuda_device), w.v_tree.to(cuda_device), mask)
            os_p, ls_p = p2p.forward(*args, seqlens_slices=sls)
            os_c, ls_c = ref.forward(*args, seqlens_slices=sls)
            torch.cuda.synchronize()
            o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, oracle_masks(w),
                                            seqlens=w.seqlens)
            Hp = H // P
            for r in range(P):
                assert torch.equal(os_p[r], os_c[r]) and torch.equal(ls_p[r], ls_c[r]), f"step {step} rank {r}"
                hs = slice(r * Hp, (r + 1) * Hp)
                compare(os_p[r], ls_p[r], o_ref[:, :, hs], l_ref[:, hs], dtype, f"p2p P={P} step {step} rank {r}")
    finally:
        p2p.close()
        ref.close()
