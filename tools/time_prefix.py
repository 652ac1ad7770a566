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


def time_prefix(name, reps=60):
    dev = torch.device("cuda:0")
    w = config_workload(name, seed=0)
    x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
    mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
    o, lse = hta.hta_forward(*x, mask)
    shape = hta.make_shape(x[0], k_cache=x[1], k_tree=x[3])
    ws = hta.new_workspace(shape, dev)
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
    for name in sys.argv[1:] or ["llama8b_64k"]:
        med, mn = time_prefix(name)
        print(f"{name}: prefix mean {med:.1f} us min {mn:.1f}", flush=True)
