"""Diagnostics: hta_forward_paged (16-key pages shuffled in a pool) vs hta_forward on the
contiguous Llama-8B-64k cache, each timed alone with CUDA events after an L2 flush (write + two
reads), median of 20.  HTA_LIB selects the library."""
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
    w = config_workload("llama8b_64k", seed=0)
    q, kc, vc, kt, vt = (t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree))
    mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
    page = int(os.environ.get("PAGE", "16"))
    maxp = w.N // page
    perm = torch.randperm(w.B * maxp, generator=torch.Generator().manual_seed(0)).view(w.B, maxp)
    if os.environ.get("NOSHUFFLE"):
        perm = torch.arange(w.B * maxp).view(w.B, maxp)
    kp = torch.empty(w.B * maxp, page, w.H_kv, w.d, dtype=kc.dtype, device=dev)
    vp = torch.empty_like(kp)
    kp[perm.to(dev).view(-1)] = kc.reshape(w.B * maxp, page, w.H_kv, w.d)
    vp[perm.to(dev).view(-1)] = vc.reshape(w.B * maxp, page, w.H_kv, w.d)
    bt = perm.to(torch.int32).to(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    f32 = flush.view(torch.float32)

    def timeit(fn):
        ts = []
        for i in range(25):
            flush.fill_(i & 0xFF)
            f32.sum()
            f32.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ts)

    tp = timeit(lambda: hta.hta_forward_paged(q, kp, vp, bt, kt, vt, mask))
    tc = timeit(lambda: hta.hta_forward(q, kc, vc, kt, vt, mask))
    print(f"page {page}{' (in order)' if os.environ.get('NOSHUFFLE') else ''}: paged {tp:.1f} us, contiguous {tc:.1f} us")


if __name__ == "__main__":
    main()
