"""Launch cost of the tree utility kernels (diagnostics): 200 back-to-back launches, mean per launch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads import accept_tokens, beam_tree  # noqa: E402

dev = torch.device("cuda:0")
par = beam_tree(64, seed=0)
dr, tg, ctx = accept_tokens(par, seed=0, vocab=32000, p_match=0.8)
par, dr, tg = par.to(dev), dr.to(dev), tg.to(dev)
mask = torch.empty(64, 64, dtype=torch.uint8, device=dev)
path = torch.empty(64, dtype=torch.int32, device=dev)
pl = torch.empty(1, dtype=torch.int32, device=dev)
bo = torch.empty(1, dtype=torch.int32, device=dev)
fns = {"mask": lambda: hta.hta_build_tree_mask(par, mask),
       "accept": lambda: hta.hta_accept_greedy(par, dr, tg, root=0, context_argmax=ctx, path=path, path_len=pl, bonus=bo),
       "tree_step": lambda: hta.hta_tree_step(par, dr, tg, root=0, context_argmax=ctx, mask=mask, path=path,
                                              path_len=pl, bonus=bo)}
for name, fn in fns.items():
    for _ in range(10):
        fn()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(200):
            fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) * 1e3 / 200:.2f} us per launch (graph, back to back)")
