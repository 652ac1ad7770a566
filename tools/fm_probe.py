"""Fused split combine on vs off (diagnostics): graph-replayed hta_forward_tree / hta_forward with
the split combine inside the prefix kernel (hta_set_fused_merge(1)) and as its own kernel (0), L2
read-flushed before each replay; median / p10 / p90 of 100 replays.

    python tools/fm_probe.py [workload ...]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads.generators import config_workload  # noqa: E402


def time_graph(fn, flush, dev, n=100):
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for i in range(n + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.sum()
        flush.sum()
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2], ts[len(ts) // 10], ts[(9 * len(ts)) // 10]


def main():
    dev = torch.device("cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev).view(torch.float32)
    for name in sys.argv[1:] or ["llama8b_64k", "longchat7b_16k", "qwq32b_32k_b4", "llama8b_128k_t128"]:
        w = config_workload(name, seed=0)
        x = {k: getattr(w, k).to(dev) for k in ("q", "k_cache", "v_cache", "k_tree", "v_tree")}
        parents = w.parents[0].to(dev)
        mask = hta.hta_build_tree_mask(parents)
        shape = hta.make_shape(x["q"], k_cache=x["k_cache"], k_tree=x["k_tree"])
        ws = hta.new_workspace(shape, dev)
        o = torch.empty_like(x["q"])
        lse = torch.empty(w.B, w.H, w.T, dtype=torch.float32, device=dev)
        args = (x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"])
        out = []
        for fm in (1, 0):
            prev = hta.set_fused_merge(bool(fm))
            for nm, fn in (("forward_tree", lambda: hta.hta_forward_tree(*args, parents, o=o, lse_out=lse, ws=ws)),
                           ("forward", lambda: hta.hta_forward(*args, mask, o=o, lse_out=lse, ws=ws))):
                med, p10, p90 = time_graph(fn, flush, dev)
                out.append(f"{nm}[fm={fm}] {med:.1f} ({p10:.1f}-{p90:.1f})")
            hta.set_fused_merge(prev)
        print(f"{name}: " + ", ".join(out), flush=True)


if __name__ == "__main__":
    main()
