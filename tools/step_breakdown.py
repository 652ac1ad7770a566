"""Where the time of one verification step goes (diagnostics; tools/, not the product).

    python tools/step_breakdown.py [workload]

Times (CUDA events, L2 flushed before each repetition, median of 20) each launch of the step on
its own, the whole step issued eagerly, and the whole step replayed from a CUDA graph.
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads import accept_tokens  # noqa: E402
from workloads.generators import config_workload  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "llama8b_64k"
    dev = torch.device("cuda:0")
    w = config_workload(name, seed=0)
    x = {k: getattr(w, k).to(dev) for k in ("q", "k_cache", "v_cache", "k_tree", "v_tree")}
    parents = w.parents[0].to(dev)
    dr, tg, ctx = accept_tokens(w.parents[0], seed=0, vocab=32000, p_match=0.8)
    dr, tg = dr.to(dev), tg.to(dev)
    T = w.T
    mask = hta.hta_build_tree_mask(parents)
    o, lse = hta.hta_forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], mask)
    shape = hta.make_shape(x["q"], k_cache=x["k_cache"], k_tree=x["k_tree"])
    wsb = hta.new_workspace(shape, dev)
    path = torch.empty(T, dtype=torch.int32, device=dev)
    plen = torch.empty(1, dtype=torch.int32, device=dev)
    bonus = torch.empty(1, dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def f_mask():
        hta.hta_build_tree_mask(parents, mask)

    def f_fwd():
        hta.hta_forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], mask, o=o, lse_out=lse, ws=wsb)

    def f_acc():
        hta.hta_accept_greedy(parents, dr, tg, root=0, context_argmax=ctx, path=path, path_len=plen, bonus=bonus)

    def f_step():
        f_mask()
        f_fwd()
        f_acc()

    def t(fn, reps=20):
        ts = []
        for i in range(reps + 3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(i & 0xFF)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ts), min(ts)

    pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(23)]
    for e in pe:
        e[0].record(), e[1].record()
    torch.cuda.synchronize()
    fl32 = flush.view(torch.float32)
    for mode in ("write-flush", "read-flush", "no-flush"):
        pre = []
        for i in range(23):
            if mode == "write-flush":
                flush.fill_(i & 0xFF)
            elif mode == "read-flush":
                fl32.sum()
            hta.hta_forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], mask, o=o, lse_out=lse,
                            ws=wsb, events=pe[i])
            torch.cuda.synchronize()
            if i >= 3:
                pre.append(pe[i][0].elapsed_time(pe[i][1]) * 1e3)
        print(f"{name}: prefix kernel alone ({mode}) median {statistics.median(pre):.1f} us min {min(pre):.1f}")
    # the same cache stored head-major ([B, H_kv, N, d]) and passed as a strided [B, N, H_kv, d] view
    khm = x["k_cache"].permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
    vhm = x["v_cache"].permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
    pre = []
    for i in range(23):
        fl32.sum()
        hta.hta_forward(x["q"], khm, vhm, x["k_tree"], x["v_tree"], mask, o=o, lse_out=lse, ws=wsb, events=pe[i])
        torch.cuda.synchronize()
        if i >= 3:
            pre.append(pe[i][0].elapsed_time(pe[i][1]) * 1e3)
    print(f"{name}: prefix kernel alone (read-flush, head-major KV) median {statistics.median(pre):.1f} us "
          f"min {min(pre):.1f}")
    del khm, vhm
    for nm, fn in (("mask", f_mask), ("forward", f_fwd), ("accept", f_acc), ("step eager", f_step)):
        med, mn = t(fn)
        print(f"  {nm:12s} median {med:7.1f} us  min {mn:7.1f}")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        f_step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f_step()
    med, mn = t(g.replay)
    print(f"  {'step graph':12s} median {med:7.1f} us  min {mn:7.1f}")
    # back-to-back (L2 warm, no flush): steady-state rate
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"  graph back-to-back (no flush): {a.elapsed_time(b) * 1e3 / 50:.1f} us/step")


if __name__ == "__main__":
    main()
