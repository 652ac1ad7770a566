"""Median time of the prefix kernel alone (CUDA events around it via hta_forward_timed, L2 read-
flushed before each launch) for one or more workloads.  Diagnostics (tools/, not the product).

    python tools/time_prefix.py [workload ...]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads.generators import config_workload  # noqa: E402


def time_prefix(name, reps=60, fp8=False):
    dev = torch.device("cuda:0")
    w = config_workload(name, seed=0)
    x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
    mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
    o, lse = hta.hta_forward(*x, mask)
    shape = hta.make_shape(x[0], k_cache=x[1], k_tree=x[3])
    ws = hta.new_workspace(shape, dev)
    if fp8:  # the prefix pass over an E4M3 cache (hta_prefix_attn_fp8kv: prefix kernel + split merge)
        from workloads import fp8_cache
        k8, ks = fp8_cache(w.k_cache)
        v8, vs = fp8_cache(w.v_cache)
        k8, v8, ks, vs = k8.to(dev), v8.to(dev), ks.to(dev), vs.to(dev)
        op = torch.empty(w.B, w.T, w.H, w.d, dtype=torch.float32, device=dev)
        lp = torch.empty(w.B, w.H, w.T, dtype=torch.float32, device=dev)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev).view(torch.float32)
        ts = []
        for i in range(reps + 3):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            flush.sum()
            flush.sum()
            ev[0].record()
            hta.hta_prefix_attn_fp8kv(x[0], k8, v8, ks, vs, o_part=op, lse_part=lp, ws=ws)
            ev[1].record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
        return statistics.mean(ts), min(ts)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev).view(torch.float32)
    ts = []
    for i in range(reps + 3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for e in ev:
            e.record()
        torch.cuda.synchronize()
        flush.sum()
        flush.sum()
        hta.hta_forward(*x, mask, o=o, lse_out=lse, ws=ws, events=ev)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    return statistics.mean(ts), min(ts)


if __name__ == "__main__":
    fp8 = os.environ.get("FP8") == "1"
    for name in sys.argv[1:] or ["llama8b_64k"]:
        med, mn = time_prefix(name, fp8=fp8)
        print(f"{name}{' fp8 prefix+merge' if fp8 else ''}: prefix mean {med:.1f} us min {mn:.1f}", flush=True)
