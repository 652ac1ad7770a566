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
    L.hta_debug_cta_times.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(16 * 2048, dtype=torch.int64, device=dev)
    hta.hta_forward(*x, mask)
    torch.cuda.synchronize()
    assert L.hta_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), cta) == 0
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    warm = int(os.environ.get("TRACE_WARM", "0"))  # back-to-back launches first (sustained load)
    for _ in range(3):
        for _ in range(warm):
            hta.hta_forward(*x, mask)
        buf.zero_()
        flush.zero_()  # cold L2, as in bench.py
        hta.hta_forward(*x, mask)
        torch.cuda.synchronize()
    times = (ctypes.c_uint64 * 4096)()
    if L.hta_debug_cta_times(times) == 0:
        n_cta = 0
        rows = []
        for i in range(1024):
            e, ls, clk, x = times[4 * i: 4 * i + 4]
            if e == 0 or x == 0:
                break
            rows.append((e, ls, clk, x))
        t0 = min(r[0] for r in rows)
        ent = [(r[0] - t0) / 1e3 for r in rows]
        pro = [(r[1] - r[0]) / 1e3 for r in rows]
        ext = [(r[3] - t0) / 1e3 for r in rows]
        mhz = [r[2] / (r[3] - r[1]) * 1e3 for r in rows]
        print(f"{len(rows)} CTAs: entry spread {max(ent):.1f} us; prologue {statistics.mean(pro):.1f} us "
              f"(max {max(pro):.1f}); exit min {min(ext):.1f} median {statistics.median(ext):.1f} max {max(ext):.1f} us; "
              f"SM clock {statistics.median(mhz):.0f} MHz")
    recs = []
    for warp, row in enumerate(buf.view(16, 2048).cpu().tolist()):
        for v in row:
            if v == 0:
                break
            v &= (1 << 64) - 1
            recs.append((v & 0xFFFFFFFF, v >> 56, (v >> 52) & 0xF, (v >> 32) & 0xFFFFF, warp))
    raw = {r[1]: r[0] for r in recs if r[1] in (50, 51, 52, 53)}
    if len(raw) == 4:
        cyc = (raw[52] - raw[50]) & 0xFFFFFFFF
        ns = (raw[53] - raw[51]) & 0xFFFFFFFF
        print(f"kernel body: {cyc} cycles in {ns / 1e3:.1f} us -> SM clock {cyc / ns * 1e3:.0f} MHz")
    recs = [r for r in recs if r[1] < 50]
    t0 = min(r[0] for r in recs)
    ev = {}
    for c, e, wg, j, warp in recs:
        ev[(e, wg, j)] = c - t0
    js = sorted({k[2] for k in ev})
    print(f"{name} cta {cta}: {len(js)} KV tiles")
    rk = 1 if cta % 2 else 0
    print("  j | half A: Srdy   max    exp   Ppub | half B: Srdy   max    exp   Ppub | mma: Sissued PVA   PVB | tma K  V")
    for j in js:
        g = lambda e, w: ev.get((e, w, j), -1)
        print(f"{j:3d} | {g(10,0):9d} {g(11,0):6d} {g(12,0):6d} {g(13,0):6d} | {g(10,1):9d} {g(11,1):6d} {g(12,1):6d} "
              f"{g(13,1):6d} | {g(21,0):8d} {g(1,0):6d} {g(1,1):6d} | {g(30,0):7d} {g(31,0):7d}")
    qs = [ev[(14, w, 0)] for w in range(8) if (14, w, 0) in ev]
    if qs:
        print(f"Q staged by softmax warps: {min(qs)}..{max(qs)}; MMA saw q_full at {ev.get((22, 0, 0), -1)}; "
              f"first K TMA {ev.get((30, 0, 0), -1)}, first S issued {ev.get((21, 0, 0), -1)}")
    # per-tile skew of P publication across the 8 softmax warps of this CTA (event 13, tag = warp - 2)
    sk = []
    for j in js:
        ts = [ev[(13, w, j)] for w in range(8) if (13, w, j) in ev]
        if len(ts) == 8:
            sk.append((j, min(ts), max(ts), [t - min(ts) for t in ts]))
    for j, a, b, rel in sk[20:26]:
        print(f"P published tile {j}: first {a} last {b} skew {b - a}  per warp {rel}")
    if sk:
        print("mean P skew across warps:", statistics.mean(b - a for _, a, b, _ in sk))
    for w in (0,):
        d = lambda a, b: [ev[(b, w, j)] - ev[(a, w, j)] for j in js if (a, w, j) in ev and (b, w, j) in ev]
        nxt = [ev[(10, w, j + 1)] - ev[(13, w, j)] for j in js if (13, w, j) in ev and (10, w, j + 1) in ev]
        if d(10, 11):
            print(f"wg{w}: ld+max {statistics.mean(d(10, 11)):.0f}  exp {statistics.mean(d(11, 12)):.0f}  "
                  f"store+arrive {statistics.mean(d(12, 13)):.0f}  P->next S {statistics.mean(nxt) if nxt else 0:.0f}")
    w = 0
    seg = lambda a, b: [ev[(b, w, j)] - ev[(a, w, j)] for j in js[2:-2] if (a, w, j) in ev and (b, w, j) in ev]
    nx = [ev[(10, w, j + 1)] - ev[(12, w, j)] for j in js[2:-2] if (12, w, j) in ev and (10, w, j + 1) in ev]
    if seg(10, 16) and seg(16, 15):
        print(f"warp 2 per tile: S wait->ld issued+publish {statistics.mean(seg(10, 16)):.0f}  ld wait "
              f"{statistics.mean(seg(16, 15)):.0f}  max {statistics.mean(seg(15, 11)):.0f}  exp "
              f"{statistics.mean(seg(11, 12)):.0f}  after exp->next S ready {statistics.mean(nx):.0f}")
    nx19 = [ev[(19, w, j + 1)] - ev[(12, w, j)] for j in js[2:-2] if (12, w, j) in ev and (19, w, j + 1) in ev]
    if nx19 and seg(19, 10):
        print(f"  exp end -> loop top {statistics.mean(nx19):.0f}; try_wait(S, already complete) "
              f"{statistics.mean(seg(19, 10)):.0f}; S ready -> publish start (fence, tail check, ld issue) "
              f"{statistics.mean([ev[(18, w, j - 1)] - ev[(10, w, j)] for j in js if (18, w, j - 1) in ev and (10, w, j) in ev]):.0f} (incl. wait::st); "
              f"wait::st done -> P arrive {statistics.mean([ev[(13, w, j)] - ev[(18, w, j)] for j in js if (13, w, j) in ev and (18, w, j) in ev]):.0f}")
    rdy = [1 for j in js if (17, 1, j) in ev]
    nrd = [1 for j in js if (17, 0, j) in ev]
    if rdy or nrd:
        print(f"S(j+1) already complete when exp(j) ends: {len(rdy)} of {len(rdy) + len(nrd)} tiles")
    tiles = [ev[(10, 0, j)] for j in js if (10, 0, j) in ev]
    if len(tiles) > 2:
        print(f"period (wg0 S ready to S ready): {(tiles[-1] - tiles[1]) / (len(tiles) - 2):.0f} cycles")


if __name__ == "__main__":
    main()
