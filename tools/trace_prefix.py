"""Pipeline timeline of one CTA of the prefix kernel (diagnostics; needs libhta_trace.so).

    python -m paper_2502_17421_b200.build --trace
    HTA_LIB=paper_2502_17421_b200/libhta_trace.so python tools/trace_prefix.py [workload]

Events (see HTA_TR in csrc/prefix_tc.cu): MMA warp 1 = p_full satisfied (PV about to issue);
softmax warp: 10 = S ready, 11 = S loaded + row max, 12 = exp loop done, 13 = P published.
"""
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HTA_LIB", os.path.join(ROOT, "paper_2502_17421_b200", "libhta_trace.so"))

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads.generators import config_workload  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "llama8b_64k"
    cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dev = torch.device("cuda:0")
    w = config_workload(name, seed=0)
    x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
    mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
    L = hta.lib()
    L.hta_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = torch.zeros(16 * 2048, dtype=torch.int64, device=dev)
    hta.hta_forward(*x, mask)
    torch.cuda.synchronize()
    assert L.hta_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), cta) == 0
    for _ in range(3):
        buf.zero_()
        hta.hta_forward(*x, mask)
        torch.cuda.synchronize()
    recs = []
    for warp, row in enumerate(buf.view(16, 2048).cpu().tolist()):
        for v in row:
            if v == 0:
                break
            v &= (1 << 64) - 1
            recs.append((v & 0xFFFFFFFF, v >> 56, (v >> 52) & 0xF, (v >> 32) & 0xFFFFF, warp))
    t0 = min(r[0] for r in recs)
    ev = {}
    for c, e, wg, j, warp in recs:
        ev[(e, wg, j)] = c - t0
    js = sorted({k[2] for k in ev})
    print(f"{name} cta {cta}: {len(js)} KV tiles")
    rk = 1 if cta % 2 else 0
    print("  j | softmax: Srdy    max    exp  pvdone  Ppub | mma: Swait  Sissued  Pseen PVissued | tma K  V")
    for j in js:
        g = lambda e, w: ev.get((e, w, j), -1)
        print(f"{j:3d} | {g(10,rk):12d} {g(11,rk):6d} {g(12,rk):6d} {g(14,rk):6d} {g(13,rk):6d} | {g(20,0):7d} "
              f"{g(21,0):7d} {g(1, j & 1):7d} {g(22,0):7d} | {g(30,0):7d} {g(31,0):7d}")
    for w in (rk,):
        d = lambda a, b: [ev[(b, w, j)] - ev[(a, w, j)] for j in js if (a, w, j) in ev and (b, w, j) in ev]
        nxt = [ev[(10, w, j + 1)] - ev[(13, w, j)] for j in js if (13, w, j) in ev and (10, w, j + 1) in ev]
        if d(10, 11):
            print(f"wg{w}: ld+max {statistics.mean(d(10, 11)):.0f}  exp {statistics.mean(d(11, 12)):.0f}  "
                  f"store+arrive {statistics.mean(d(12, 13)):.0f}  P->next S {statistics.mean(nxt) if nxt else 0:.0f}")
    tiles = [ev[(10, rk, j)] for j in js if (10, rk, j) in ev]
    if len(tiles) > 2:
        print(f"period (wg0 S ready to S ready): {(tiles[-1] - tiles[1]) / (len(tiles) - 2):.0f} cycles")


if __name__ == "__main__":
    main()
