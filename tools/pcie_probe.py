"""PCIe copy costs of the end-to-end step's pieces (diagnostics): graph-captured pinned copies,
mean of 50 replays each."""
import statistics

import torch

dev = torch.device("cuda:0")
res = {}
for nm, n, h2d in (("q+tokens H2D 512KiB", 513 * 1024, True), ("tree K/V H2D 256KiB", 256 * 1024, True),
                   ("all inputs H2D 768KiB", 769 * 1024, True), ("O+path D2H 512KiB", 513 * 1024, False)):
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    devb = torch.empty(n, dtype=torch.uint8, device=dev)
    fn = (lambda: devb.copy_(host, non_blocking=True)) if h2d else (lambda: host.copy_(devb, non_blocking=True))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for i in range(53):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    res[nm] = statistics.mean(ts)
print({k: round(v, 1) for k, v in res.items()})
