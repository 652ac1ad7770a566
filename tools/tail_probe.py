"""Where the verification step's time goes outside the prefix kernel (diagnostics).

    python tools/tail_probe.py [workload]

Each variant is captured as a CUDA graph and replayed with the L2 read-flushed before each replay
(median of 30, CUDA events around the replay):
  prefix      the prefix kernel alone (events inside hta_forward_timed, eager)
  forward     hta_forward (prefix + tree/merge kernels)
  mask+fwd    a0 mask kernel, then hta_forward
  step        a0 + hta_forward, a6 accept on a forked stream (bench.py's step)
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
    mask = hta.hta_build_tree_mask(parents)
    o, lse = hta.hta_forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], mask)
    shape = hta.make_shape(x["q"], k_cache=x["k_cache"], k_tree=x["k_tree"])
    wsb = hta.new_workspace(shape, dev)
    path = torch.empty(w.T, dtype=torch.int32, device=dev)
    plen = torch.empty(1, dtype=torch.int32, device=dev)
    bonus = torch.empty(1, dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev).view(torch.float32)
    side = torch.cuda.Stream(device=dev)

    def fwd(events=None):
        hta.hta_forward(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], mask, o=o, lse_out=lse, ws=wsb,
                        events=events)

    def mask_fwd():
        hta.hta_build_tree_mask(parents, mask)
        fwd()

    def step():
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            hta.hta_accept_greedy(parents, dr, tg, root=0, context_argmax=ctx, path=path, path_len=plen, bonus=bonus)
        mask_fwd()
        cur.wait_stream(side)

    def acc():
        hta.hta_accept_greedy(parents, dr, tg, root=0, context_argmax=ctx, path=path, path_len=plen, bonus=bonus)

    def step_acc_first():
        acc()
        mask_fwd()

    def step_acc_last():
        mask_fwd()
        acc()

    def step_side_after_mask():
        cur = torch.cuda.current_stream()
        hta.hta_build_tree_mask(parents, mask)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            acc()
        fwd()
        cur.wait_stream(side)

    def fwd_tree():
        hta.hta_forward_tree(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], parents, o=o, lse_out=lse,
                             ws=wsb)

    def tstep():
        hta.hta_tree_step(parents, dr, tg, root=0, context_argmax=ctx, mask=mask, path=path, path_len=plen,
                          bonus=bonus)

    def bench_step():  # bench.py's step: a0 + a6 forked beside hta_forward_tree
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            tstep()
        fwd_tree()
        cur.wait_stream(side)

    def tstep_then_fwd_tree():
        tstep()
        fwd_tree()

    def fused_step():
        hta.hta_tree_step(parents, dr, tg, root=0, context_argmax=ctx, mask=mask, path=path, path_len=plen,
                          bonus=bonus)
        fwd()

    def graph(fn):
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    def t(fn, reps=100):
        ts = []
        for i in range(reps + 3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.sum()
            flush.sum()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        return statistics.mean(ts)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(33)]
    for a, b in ev:
        a.record()
        b.record()
    torch.cuda.synchronize()
    pre = []
    for i in range(33):
        flush.sum()
        flush.sum()
        fwd(ev[i])
        torch.cuda.synchronize()
        if i >= 3:
            pre.append(ev[i][0].elapsed_time(ev[i][1]) * 1e3)
    res = {"prefix": statistics.mean(pre)}
    for nm, fn in (("forward", fwd), ("mask+fwd", mask_fwd), ("step", step), ("accept", acc),
                   ("acc;mask;fwd", step_acc_first), ("mask;fwd;acc", step_acc_last),
                   ("mask;(acc|fwd)", step_side_after_mask), ("tree_step;fwd", fused_step),
                   ("fwd_tree", fwd_tree), ("tree_step", tstep), ("tree_step|fwd_tree", bench_step),
                   ("tree_step;fwd_tree", tstep_then_fwd_tree)):
        res[nm] = t(graph(fn).replay)
    print(name + ": " + ", ".join(f"{k} {v:.1f} us" for k, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
