import statistics, torch, sys
sys.path.insert(0, "/root/repo")
from paper_2502_17421_b200 import hta
from workloads.generators import config_workload
dev = torch.device("cuda:0")
w = config_workload("qwq32b_32k_b4", seed=0)
x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev).view(torch.float32)
for ns in (0, 1, 2, 3, 4):
    ts = []
    for i in range(13):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for e in ev: e.record()
        torch.cuda.synchronize()
        flush.sum()
        hta.hta_forward(*x, mask, num_splits=ns, events=ev)
        torch.cuda.synchronize()
        if i >= 3: ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    print("num_splits", ns, "prefix us", round(statistics.median(ts), 1))
