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
    fwd = lambda: hta.hta_forward(*x, mask)  # noqa: E731
    if os.environ.get("PAGED"):  # the paged forward over in-order 16-key pages
        page = 16
        maxp = w.N // page
        kp = x[1].reshape(w.B * maxp, page, w.H_kv, w.d).contiguous()
        vp = x[2].reshape(w.B * maxp, page, w.H_kv, w.d).contiguous()
        bt = torch.arange(w.B * maxp, dtype=torch.int32, device=dev).view(w.B, maxp)
        fwd = lambda: hta.hta_forward_paged(x[0], kp, vp, bt, x[3], x[4], mask)  # noqa: E731
    L = hta.lib()
    L.hta_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.hta_debug_cta_times.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(32 * 2048, dtype=torch.int64, device=dev)
    fwd()
    torch.cuda.synchronize()
    assert L.hta_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), cta) == 0
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    warm = int(os.environ.get("TRACE_WARM", "0"))  # back-to-back launches first (sustained load)
    for _ in range(3):
        for _ in range(warm):
            fwd()
        buf.zero_()
        flush.zero_()  # cold L2, as in bench.py
        fwd()
        torch.cuda.synchronize()
    times = (ctypes.c_uint64 * 8192)()
    if L.hta_debug_cta_times(times) == 0:
        n_cta = 0
        rows = []
        for i in range(1024):
            e, ls, clk, x = times[4 * i: 4 * i + 4]  # g_cta_times[1024][4] (prefix_tc.cu)
            if e == 0 or x == 0:
                break
            rows.append((e, ls, clk, x))
        t0 = min(r[0] for r in rows)
        ent = [(r[0] - t0) / 1e3 for r in rows]
        pro = [(r[1] - r[0]) / 1e3 for r in rows]
        ext = [(r[3] - t0) / 1e3 for r in rows]
        mhz = [r[2] / (r[3] - r[1]) * 1e3 for r in rows]
        slow = sorted(range(len(rows)), key=lambda i: -ext[i])[:12]
        print("slowest CTAs (blockIdx: exit us):", ", ".join(f"{i}:{ext[i]:.1f}" for i in slow))
        print(f"{len(rows)} CTAs: entry spread {max(ent):.1f} us; prologue {statistics.mean(pro):.1f} us "
              f"(max {max(pro):.1f}); exit min {min(ext):.1f} median {statistics.median(ext):.1f} max {max(ext):.1f} us; "
              f"SM clock {statistics.median(mhz):.0f} MHz")
        q = sorted(ext)
        print("exit quantiles (us): " + " ".join(f"p{p}={q[min(len(q) - 1, len(q) * p // 100)]:.1f}"
                                               for p in (10, 25, 50, 75, 90, 100)))
    recs = []
    for warp, row in enumerate(buf.view(32, 2048).cpu().tolist()):
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
    print("   j | K issued  K landed  S issued | S ready  max   exp | P all pub | V issued  V landed  P seen(PV) | K lat  V lat")
    rows = []
    for j in js:
        g = lambda e, w=0: ev.get((e, w, j), -1)
        pub = [ev[(13, w, j)] for w in range(16) if (13, w, j) in ev]
        pm = max(pub) if pub else -1
        rows.append((j, g(30), g(23), g(21), g(10), g(11), g(12), pm, g(31), g(24), g(1)))
        print(f"{j:4d} | {g(30):8d} {g(23):8d} {g(21):8d} | {g(10):8d} {g(11)-g(10):5d} {g(12)-g(11):5d} | {pm:8d} | "
              f"{g(31):8d} {g(24):8d} {g(1):8d} | {g(23)-g(30):5d} {g(24)-g(31):5d}")
    mid = rows[3:-3] if len(rows) > 8 else rows
    if len(mid) > 2:
        per = (mid[-1][4] - mid[0][4]) / (len(mid) - 1)
        print(f"period (S ready to S ready, middle tiles): {per:.0f} cycles")
        wait_k = statistics.mean(max(0, r[2] - r[7 - 0] if False else 0) for r in mid)
        kl = statistics.mean(r[2] - r[1] for r in mid)
        vl = statistics.mean(r[9] - r[8] for r in mid)
        print(f"mean TMA latency (issue -> MMA warp sees full): K {kl:.0f}  V {vl:.0f} cycles")
        # what gated each PV issue: the later of V landed and P published
        gate_p = sum(1 for r in mid if r[10] - r[9] > 50)
        print(f"PV gated by P publication on {gate_p} of {len(mid)} tiles (else by V data)")
        print(" warp sm  SMSP  S->max  max->exp  exp->pub(next tile)  pub lag vs earliest warp")
        jm = [r[0] for r in mid]
        for w in range(16):
            a = [ev[(11, w, j)] - ev[(10, w, j)] for j in jm if (11, w, j) in ev and (10, w, j) in ev]
            b = [ev[(12, w, j)] - ev[(11, w, j)] for j in jm if (12, w, j) in ev and (11, w, j) in ev]
            c = [ev[(13, w, j)] - ev[(12, w, j)] for j in jm if (13, w, j) in ev and (12, w, j) in ev]
            lag = [ev[(13, w, j)] - min(ev[(13, x, j)] for x in range(16) if (13, x, j) in ev) for j in jm
                   if (13, w, j) in ev]
            if a:
                print(f"  {w:3d}  {(w + 3) % 4:3d}  {statistics.mean(a):6.0f}  {statistics.mean(b):7.0f}  "
                      f"{statistics.mean(c) if c else 0:10.0f}  {statistics.mean(lag) if lag else 0:10.0f}")
        sm = statistics.mean(r[5] - r[4] for r in mid)
        se = statistics.mean(r[6] - r[5] for r in mid)
        print(f"softmax warp 0: S ready -> max {sm:.0f}, max -> exp done {se:.0f}")


if __name__ == "__main__":
    main()
