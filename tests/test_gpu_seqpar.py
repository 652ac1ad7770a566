"""hta_forward_seqpar on the GPU with a one-rank NCCL communicator (the only world size a single
B200 allows): the local split-KV pass combined into one destination-major partial, the NCCL
exchange (self copy), and the final merge with the tree pass -- vs the fp64 oracle, with and
without the output all-gather.  The P = 2 data flow is covered on CPU by test_seqpar_gloo.py."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload

from gpu_util import compare, oracle_masks, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(cuda_device):
    try:
        c = hta.HtaComm(0, 1)
    except hta.HtaError as e:
        pytest.fail(f"NCCL communicator: {e}")
    yield c
    c.close()


@pytest.mark.parametrize("gather", [False, True])
@pytest.mark.parametrize("case", [(1, 64, 32, 8, 128, 3000, "beam"), (2, 13, 8, 2, 128, 1000, "random"),
                                  (1, 9, 6, 2, 64, 700, "star")])
def test_seqpar_one_rank_vs_oracle(cuda_device, comm, case, gather):
    B, T, H, Hkv, d, N, tree = case
    w = make_workload(B, T, H, Hkv, d, N, "bf16", dist="V1", seed=5, tree=tree)
    mask = oracle_masks(w)
    x = to_dev(w, cuda_device)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask, seqlens=w.seqlens)
    o, l = comm.forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], torch.from_numpy(mask).to(cuda_device),
                        cache_seqlens_local=x["sl"], gather_output=gather)
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", f"seqpar P=1 gather={gather}")


def test_seqpar_step_in_cuda_graph(cuda_device, comm):
    """The sequence-parallel step (prefix -> split combine -> NCCL exchange -> merge) captured as a
    CUDA graph (NCCL supports stream capture) replays to the eager result, bit for bit."""
    w = make_workload(1, 64, 32, 8, 128, 4000, "bf16", dist="V1", seed=8, tree="beam")
    mask = torch.from_numpy(oracle_masks(w)).to(cuda_device)
    x = to_dev(w, cuda_device)
    o_e, l_e = comm.forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask, cache_seqlens_local=x["sl"],
                            gather_output=True)
    torch.cuda.synchronize()
    o = torch.zeros_like(o_e)
    lse = torch.zeros_like(l_e)
    shape = hta.make_shape(x["q"], k_cache=x["kc"], k_tree=x["kt"])
    ws = torch.empty(comm.workspace_size(shape), dtype=torch.uint8, device=cuda_device)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        comm.forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask, cache_seqlens_local=x["sl"], gather_output=True,
                     o=o, lse_out=lse, ws=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        comm.forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask, cache_seqlens_local=x["sl"], gather_output=True,
                     o=o, lse_out=lse, ws=ws)
    o.zero_()
    lse.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o, o_e) and torch.equal(lse, l_e)
    assert not comm.async_error()


@pytest.mark.parametrize("gather", [False, True])
def test_seqpar_tree_from_parents(cuda_device, comm, gather):
    """hta_forward_seqpar_tree (the tree as its parent array; the final merge walks it) is
    bit-identical to hta_forward_seqpar over the mask hta_build_tree_mask writes, per-batch trees."""
    w = make_workload(2, 40, 8, 2, 128, 1500, "bf16", dist="V1", seed=12, tree="random")
    x = to_dev(w, cuda_device)
    par = torch.stack([w.parents[b] for b in range(2)]).to(torch.int32).to(cuda_device)
    mask = torch.stack([hta.hta_build_tree_mask(par[b]) for b in range(2)])
    o_m, l_m = comm.forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask, cache_seqlens_local=x["sl"],
                            gather_output=gather)
    o_p, l_p = comm.forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], cache_seqlens_local=x["sl"],
                            gather_output=gather, parents=par)
    torch.cuda.synchronize()
    assert torch.equal(o_m, o_p) and torch.equal(l_m, l_p)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, oracle_masks(w), seqlens=w.seqlens)
    compare(o_p, l_p, o_ref, l_ref, "bf16", "seqpar_tree P=1")


def test_seqpar_peer_memory_exchange_graph_replays(cuda_device, comm):
    """The peer-memory exchange on a real (one-rank) communicator, with the IPC export/open of
    hta_comm_p2p_alloc/open, inside a CUDA graph: the device-side step counter advances on every
    replay (alternating receive-buffer halves, flags compared with it), and every replay on new
    inputs equals the NCCL-exchange step of the reference communicator bit for bit."""
    p2p = hta.HtaComm(0, 1)
    try:
        w0 = make_workload(1, 64, 32, 8, 128, 3000, "bf16", dist="V1", seed=60, tree="beam")
        x = {k: getattr(w0, k).to(cuda_device) for k in ("q", "k_cache", "v_cache", "k_tree", "v_tree")}
        par = w0.parents[0].to(torch.int32).to(cuda_device)
        shape = hta.make_shape(x["q"], k_cache=x["k_cache"], k_tree=x["k_tree"])
        assert p2p.enable_p2p([shape])
        o = torch.empty_like(x["q"])
        lse = torch.empty(1, 32, 64, dtype=torch.float32, device=cuda_device)
        ws = torch.empty(p2p.workspace_size(shape), dtype=torch.uint8, device=cuda_device)

        def fwd():
            p2p.forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], o=o, lse_out=lse, ws=ws,
                        parents=par)

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fwd()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fwd()
        for step in range(4):
            w = make_workload(1, 64, 32, 8, 128, 3000, "bf16", dist="V1", seed=61 + step, tree="beam")
            for k in x:
                x[k].copy_(getattr(w, {"q": "q", "k_cache": "k_cache", "v_cache": "v_cache", "k_tree": "k_tree",
                                       "v_tree": "v_tree"}[k]))
            par.copy_(w.parents[0].to(torch.int32))
            g.replay()
            o_ref, l_ref = comm.forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], parents=par)
            torch.cuda.synchronize()
            assert torch.equal(o, o_ref) and torch.equal(lse, l_ref), f"replay {step}"
    finally:
        p2p.close()
