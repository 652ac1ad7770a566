"""Fused vs unfused tree pass (diagnostics): graph-replayed hta_forward (tree tiles in the prefix
kernel), hta_forward with a tree_ready event (tree pass in the tree/merge kernel) and the prefix
pass alone (hta_prefix_attn), L2 read-flushed before each replay, mean of 100.

    [HTA_LIB=...] python tools/fuse_probe.py [workload ...]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads.generators import config_workload  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev).view(torch.float32)
    for name in sys.argv[1:] or ["llama8b_64k"]:
        w = config_workload(name, seed=0)
        x = {k: getattr(w, k).to(dev) for k in ("q", "k_cache", "v_cache", "k_tree", "v_tree")}
        mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
        shape = hta.make_shape(x["q"], k_cache=x["k_cache"], k_tree=x["k_tree"])
        ws = hta.new_workspace(shape, dev)
        o = torch.empty_like(x["q"])
        lse = torch.empty(w.B, w.H, w.T, dtype=torch.float32, device=dev)
        op = torch.empty(w.B, w.T, w.H, w.d, dtype=torch.float32, device=dev)
        ready = torch.cuda.Event()
        evs = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        parents = w.parents[0].to(dev)
        args = (x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"], mask)
        fns = {
            "fused": lambda: hta.hta_forward(*args, o=o, lse_out=lse, ws=ws),
            "unfused": lambda: (ready.record(), hta.hta_forward(*args, o=o, lse_out=lse, ws=ws, tree_ready=ready)),
            "prefix_attn": lambda: hta.hta_prefix_attn(x["q"], x["k_cache"], x["v_cache"], o_part=op, lse_part=lse,
                                                       ws=ws),
            "forward_tree": lambda: hta.hta_forward_tree(x["q"], x["k_cache"], x["v_cache"], x["k_tree"], x["v_tree"],
                                                         parents, o=o, lse_out=lse, ws=ws),
            "timed(events)": lambda: hta.hta_forward(*args, o=o, lse_out=lse, ws=ws, events=evs),
        }
        if os.environ.get("FP8"):  # the forward over an E4M3 copy of the cache
            from workloads import fp8_cache
            k8, ks = fp8_cache(w.k_cache)
            v8, vs = fp8_cache(w.v_cache)
            k8, v8, ks, vs = k8.to(dev), v8.to(dev), ks.to(dev), vs.to(dev)
            fns = {"fp8": lambda: hta.hta_forward_fp8kv(x["q"], k8, v8, ks, vs, x["k_tree"], x["v_tree"], mask, o=o,
                                                        lse_out=lse),
                   "bf16": fns["fused"]}
        res = {}
        for nm, fn in fns.items():
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
            for i in range(103):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                flush.sum()
                flush.sum()
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                if i >= 3:
                    ts.append(a.elapsed_time(b) * 1e3)
            res[nm] = statistics.mean(ts)
        print(f"{name} [{os.path.basename(hta.lib()._name)}]: " + ", ".join(f"{k} {v:.1f} us" for k, v in res.items()),
              flush=True)


if __name__ == "__main__":
    main()
