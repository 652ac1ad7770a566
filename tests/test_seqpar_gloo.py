"""Sequence-parallel data flow (row a5 of SURVEY.md §8) with world size 2 over gloo, on CPU.

Each rank plays one GPU of hta_forward_seqpar: it holds the contiguous KV shard
`hta.shard_bounds(N, P, r)`, computes the prefix partial of every head over its shard (the fp64
oracle stands in for the local split-KV pass), sends head slice [p*H/P, (p+1)*H/P) to rank p (the
destination-major exchange, here an all_gather over gloo), and merges the P received prefix
partials with the tree partial of its own heads (PAPER.md:207-218 applied P+1 ways,
Appendix C).  The gathered result must equal one-shot attention over the whole
prefix + tree.  Also checks the unique-id broadcast of hta.HtaComm when NCCL is loadable.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, T, H, Hkv, d, N, seqlen = case
        w = make_workload(B, T, H, Hkv, d, N, "bf16", dist="V1", seed=21, tree="beam")
        seqlens = torch.full((B,), seqlen, dtype=torch.int32)
        mask = np.stack([oracle.tree_mask(w.parents[b]) for b in range(B)])
        lo, hi = hta.shard_bounds(N, world, rank)
        # local prefix partial over this rank's shard, all heads (valid length clamped per shard)
        sl_local = torch.clamp(seqlens - lo, 0, hi - lo).to(torch.int32)
        o_c, l_c = oracle.attention(w.q, w.k_cache[:, lo:hi], w.v_cache[:, lo:hi], w.k_tree, w.v_tree, mask,
                                    seqlens=sl_local, part="cache")
        Hp = H // world
        # destination-major blocks: block p = heads [p*Hp, (p+1)*Hp) -> rank p
        send = torch.from_numpy(np.concatenate([o_c[:, :, p * Hp:(p + 1) * Hp].reshape(-1) for p in range(world)] +
                                               [l_c[:, p * Hp:(p + 1) * Hp].reshape(-1) for p in range(world)]))
        gathered = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(gathered, send)
        no = B * T * Hp * d
        nl = B * Hp * T
        parts = []
        for src in range(world):  # what rank `src` sent to this rank
            buf = gathered[src].numpy()
            o_p = buf[rank * no:(rank + 1) * no].reshape(B, T, Hp, d)
            l_p = buf[world * no + rank * nl:world * no + (rank + 1) * nl].reshape(B, Hp, T)
            parts.append((o_p, l_p))
        o_t, l_t = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, part="tree")
        hs = slice(rank * Hp, (rank + 1) * Hp)
        parts.append((o_t[:, :, hs], l_t[:, hs]))
        # the merge folds over [B,T,Hp,d] / [B,T,Hp] layouts: LSE to [B,T,Hp] first
        o_m, l_m = oracle.merge([(o, np.transpose(l, (0, 2, 1))) for o, l in parts])
        res = torch.from_numpy(np.concatenate([o_m.reshape(-1), np.transpose(l_m, (0, 2, 1)).reshape(-1)]))
        outs = [torch.empty_like(res) for _ in range(world)]
        dist.all_gather(outs, res)
        if rank == 0:
            o_full = np.concatenate([o.numpy()[:B * T * Hp * d].reshape(B, T, Hp, d) for o in outs], axis=2)
            l_full = np.concatenate([o.numpy()[B * T * Hp * d:].reshape(B, Hp, T) for o in outs], axis=1)
            o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=seqlens)
            out_q.put((float(np.abs(o_full - o_ref).max()), float(np.abs(l_full - l_ref).max())))
        # HtaComm's unique id travels over the process group (rank 0 -> all)
        try:
            comm_uid = None
            lib = hta.lib()
            import ctypes
            buf = (ctypes.c_uint8 * 128)()
            if rank == 0 and lib.hta_comm_unique_id(buf) == 0:
                comm_uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
            flag = torch.tensor([1 if comm_uid is not None else 0])
            dist.broadcast(flag, src=0)
            if int(flag) == 1:
                uid = comm_uid if rank == 0 else torch.zeros(128, dtype=torch.uint8)
                dist.broadcast(uid, src=0)
                ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(ids, uid)
                if rank == 0:
                    out_q.put(("uid", all(torch.equal(ids[0], x) for x in ids), int(ids[0].sum())))
            elif rank == 0:
                out_q.put(("uid", None, 0))
        except (ImportError, OSError):
            if rank == 0:
                out_q.put(("uid", None, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(1, 16, 8, 2, 64, 700, 700), (2, 9, 4, 4, 64, 513, 300)])
def test_seqpar_two_ranks_gloo(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0, "seqpar gloo worker failed"
    err_o, err_l = q.get(timeout=10)
    assert err_o < 1e-12 and err_l < 1e-12, (err_o, err_l)
    tag, same, total = q.get(timeout=10)
    assert tag == "uid"
    if same is not None:
        assert same and total > 0
