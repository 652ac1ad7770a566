"""hta_commit_kv (SPEC commit_kv S:212-220) vs oracle.commit_kv:
bit-exact (a copy), for bf16 and fp32, batch > 1, the device path of hta_accept_greedy, empty
paths, saturation at N_max, strided (head-major) caches and in-place seqlens update."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import accept_tokens, make_workload

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,head_major", [("bf16", False), ("fp32", False), ("bf16", True)])
def test_commit_kv_bit_exact(cuda_device, dtype, head_major):
    B, T, H, Hkv, d, N = 3, 40, 8, 4, 128, 500
    w = make_workload(B, T, H, Hkv, d, N, dtype, dist="V0", seed=9, tree="beam")
    rng = np.random.default_rng(4)
    n0 = np.array([100, 490, 7], np.int32)  # batch 1 saturates at N_max = 500
    paths = np.zeros((B, T), np.int32)
    lens = np.zeros(B, np.int32)
    for b in range(B):
        par = w.parents[b].tolist()
        leaf = int(rng.integers(1, T))
        chain = [leaf]
        while par[chain[-1]] >= 0:
            chain.append(par[chain[-1]])
        path = chain[::-1]
        paths[b, :len(path)] = path
        lens[b] = len(path)
    lens[2] = 0  # empty acceptance
    k_ref, v_ref, n_ref = oracle.commit_kv(w.k_cache.float().numpy(), w.v_cache.float().numpy(), n0,
                                           w.k_tree.float().numpy(), w.v_tree.float().numpy(), paths, lens)
    dev = cuda_device
    if head_major:  # [B, H_kv, N, d] storage seen as a strided [B, N, H_kv, d] view
        kc = w.k_cache.permute(0, 2, 1, 3).contiguous().to(dev).permute(0, 2, 1, 3)
        vc = w.v_cache.permute(0, 2, 1, 3).contiguous().to(dev).permute(0, 2, 1, 3)
    else:
        kc, vc = w.k_cache.to(dev), w.v_cache.to(dev)
    sl = torch.from_numpy(n0).to(dev)
    hta.hta_commit_kv(torch.from_numpy(paths).to(dev), torch.from_numpy(lens).to(dev), w.k_tree.to(dev),
                      w.v_tree.to(dev), kc, vc, sl, seqlens_out=sl)  # in place
    torch.cuda.synchronize()
    assert sl.cpu().tolist() == n_ref.tolist()
    assert np.array_equal(kc.float().cpu().numpy(), k_ref)
    assert np.array_equal(vc.float().cpu().numpy(), v_ref)


def test_commit_after_device_accept(cuda_device):
    """The accept -> commit chain stays on the device: hta_accept_greedy's path and length feed
    hta_commit_kv directly."""
    B, T, H, Hkv, d, N = 1, 64, 32, 8, 128, 4096
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist="V1", seed=2, tree="beam")
    par = w.parents[0]
    draft, tgt, ctx = accept_tokens(par, seed=3, vocab=32000, p_match=0.9)
    path_h, bonus_h = oracle.accept_greedy(par, draft, tgt, root=0)
    dev = cuda_device
    path, plen, bonus = hta.hta_accept_greedy(par.to(dev), draft.to(dev), tgt.to(dev), root=0)
    n0 = np.array([3000], np.int32)
    kc, vc = w.k_cache.to(dev), w.v_cache.to(dev)
    sl = torch.from_numpy(n0).to(dev)
    out = hta.hta_commit_kv(path, plen, w.k_tree.to(dev), w.v_tree.to(dev), kc, vc, sl)
    torch.cuda.synchronize()
    paths = np.zeros((1, T), np.int32)
    paths[0, :len(path_h)] = path_h
    k_ref, v_ref, n_ref = oracle.commit_kv(w.k_cache.float().numpy(), w.v_cache.float().numpy(), n0,
                                           w.k_tree.float().numpy(), w.v_tree.float().numpy(), paths, [len(path_h)])
    assert out.cpu().tolist() == n_ref.tolist() and len(path_h) >= 2
    assert np.array_equal(kc.float().cpu().numpy(), k_ref)
    assert np.array_equal(vc.float().cpu().numpy(), v_ref)


def test_commit_negative_seqlen_counts_as_empty(cuda_device):
    """A negative committed length is clamped to 0 (no write before row 0): the rows land at
    0..len-1, like the oracle's commit onto an empty cache."""
    B, T, H, Hkv, d, N = 2, 8, 4, 2, 64, 64
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist="V0", seed=6, tree="chain")
    paths = np.tile(np.arange(T, dtype=np.int32), (B, 1))
    lens = np.array([3, 5], np.int32)
    n0 = np.array([-7, 10], np.int32)
    k_ref, v_ref, n_ref = oracle.commit_kv(w.k_cache.float().numpy(), w.v_cache.float().numpy(),
                                           np.maximum(n0, 0), w.k_tree.float().numpy(), w.v_tree.float().numpy(),
                                           paths, lens)
    dev = cuda_device
    kc, vc = w.k_cache.to(dev), w.v_cache.to(dev)
    out = hta.hta_commit_kv(torch.from_numpy(paths).to(dev), torch.from_numpy(lens).to(dev), w.k_tree.to(dev),
                            w.v_tree.to(dev), kc, vc, torch.from_numpy(n0).to(dev))
    torch.cuda.synchronize()
    assert out.cpu().tolist() == n_ref.tolist() == [3, 15]
    assert np.array_equal(kc.float().cpu().numpy(), k_ref)
    assert np.array_equal(vc.float().cpu().numpy(), v_ref)
