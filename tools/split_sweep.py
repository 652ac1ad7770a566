"""Time hta_forward of a workload with forced split counts (diagnostics for the planner in
csrc/hta_api.cu).  usage: python tools/split_sweep.py WORKLOAD S1 S2 ...   (0 = planner's choice)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads.generators import config_workload  # noqa: E402


def main():
    name = sys.argv[1]
    dev = torch.device("cuda:0")
    w = config_workload(name, seed=0)
    x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
    mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for S in [int(a) for a in sys.argv[2:]]:
        ts = []
        for it in range(13):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hta.hta_forward(*x, mask, num_splits=S)
            e1.record()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"{name} splits={S}: forward median {ts[len(ts) // 2]:.1f} us  min {ts[0]:.1f} us")


if __name__ == "__main__":
    main()
