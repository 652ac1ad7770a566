"""Pipeline timeline of one CTA of the prefix kernel (diagnostics; needs libhta_trace.so).

    python -m paper_2502_17421_b200.build --trace
    HTA_LIB=paper_2502_17421_b200/libhta_trace.so python tools/trace_prefix.py [workload] [cta]

Events (HTA_TR in csrc/prefix_tc.cu), per warp, clock64 cycles:
  MMA warp 1:  2 = K_j landed, S_j issue   3 = V_j landed   1 = P_j published, PV_j issue
  producers:   30 = K slot j free, TMA issued (warp 0)   31 = V slot j (warp 2)
  softmax:     10 = S_j ready   11 = S_j loaded   12 = exponentials done   13 = hand-over of
               tile j-1 read   15 = P_j stores landed   14 = P_j published
  all warps:   0 = kernel entry   63 = exit
"""
import ctypes
import os
import statistics
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HTA_LIB", os.path.join(ROOT, "paper_2502_17421_b200", "libhta_trace.so"))

import torch  # noqa: E402

from paper_2502_17421_b200 import hta  # noqa: E402
from workloads.generators import config_workload  # noqa: E402

RECS = 1024


def analyze_t8(ev, rel, name, cta):
    """prefix_t8.cu events: TMA 40/41 (K/V slot free, issue); K widening 42 landed, 43 TMEM buffer
    free, 44 done; V 45/46/47; MMA 48 S_j issue, 49 PV_j issue; softmax 50 S ready, 51 pass 1
    done, 52 vote done, 53 published."""
    med = lambda xs: statistics.median(xs) if xs else 0  # noqa: E731
    exit_t = max(rel(v[0]) for (wi, e), v in ev.items() if e == 0)
    print(f"{name} CTA {cta} (transposed FP8 kernel): last warp entry at {exit_t}")
    mma = next((w for w in range(32) if (w, 49) in ev), None)
    if mma is None:
        print("no MMA records")
        return
    pv, sis = ev[(mma, 49)], ev[(mma, 48)]
    js = sorted(pv)
    per = [pv[b] - pv[a] for a, b in zip(js, js[1:])]
    print(f"MMA warp {mma}: {len(js)} PV; first PV at {rel(pv[js[0]])}, last at {rel(pv[js[-1]])}; "
          f"period median {med(per):.0f} (p10 {sorted(per)[len(per) // 10] if per else 0}, "
          f"p90 {sorted(per)[9 * len(per) // 10] if per else 0})")
    tw = next((w for w in range(32) if (w, 40) in ev), None)
    if tw is not None:
        kw_ = next((w for w in range(32) if (w, 42) in ev), None)
        vw_ = next((w for w in range(32) if (w, 45) in ev), None)
        for nm, ei, wl, el in (("K", 40, kw_, 42), ("V", 41, vw_, 45)):
            if wl is None or (tw, ei) not in ev:
                continue
            a, b_ = ev[(tw, ei)], ev[(wl, el)]
            jj = sorted(j for j in a if j in b_)
            print(f"{nm} TMA issue -> landed (seen by its widening warp) median {med([b_[j] - a[j] for j in jj]):.0f}; "
                  f"issue lead over PV_j {med([pv[j] - a[j] for j in jj if j in pv]):.0f}")
    s_iss = [ev[(mma, 55)][j] - sis[j] for j in sorted(ev.get((mma, 55), {})) if j in sis]
    pv_iss = [ev[(mma, 56)][j] - pv[j] for j in sorted(ev.get((mma, 56), {})) if j in pv]
    print(f"MMA issue durations: S batch {med(s_iss):.0f}, PV batch {med(pv_iss):.0f} cycles (median)")
    for nm, evs in (("K", (42, 43, 44)), ("V", (45, 45, 47))):
        for w in (w for w in range(32) if (w, evs[2]) in ev):
            a, b_, c_ = (ev.get((w, e), {}) for e in evs)
            jj = sorted(j for j in c_ if j in a and j in b_)
            print(f"{nm} warp {w}: landed->buffer free {med([b_[j] - a[j] for j in jj]):.0f}, "
                  f"widen {med([c_[j] - b_[j] for j in jj]):.0f}, done->next landed "
                  f"{med([a[j2] - c_[j1] for j1, j2 in zip(jj, jj[1:])]):.0f}")
    sm = [w for w in range(32) if (w, 53) in ev]
    for w in sm:
        e0, e1, e2, e3 = (ev.get((w, e), {}) for e in (50, 51, 52, 53))
        jj = sorted(j for j in e3 if j in e0 and j in e1 and j in e2)
        idle = [e0[j2] - e3[j1] for j1, j2 in zip(jj, jj[1:])]
        print(f"softmax warp {w}: pass1 {med([e1[j] - e0[j] for j in jj]):.0f}, vote {med([e2[j] - e1[j] for j in jj]):.0f}, "
              f"->published {med([e3[j] - e2[j] for j in jj]):.0f}, idle waiting for S {med(idle):.0f}")
    print("tile: S_j issued | S_j ready (w0) | published (all softmax warps) | PV_j issued | K_j done | V_j done  (cycles)")
    for j in js[max(0, len(js) // 2 - 5):len(js) // 2 + 5]:
        pubs = [ev.get((w, 53), {}).get(j) for w in sm]
        pubs = [rel(x) for x in pubs if x is not None]
        kd = [ev.get((w, 44), {}).get(j) for w in range(32)]
        vd = [ev.get((w, 47), {}).get(j) for w in range(32)]
        kd = max(rel(x) for x in kd if x is not None) if any(x is not None for x in kd) else "-"
        vd = max(rel(x) for x in vd if x is not None) if any(x is not None for x in vd) else "-"
        sr = ev.get((0, 50), {}).get(j)
        print(f"{j:4d}: {rel(sis[j]) if j in sis else '-'} | {rel(sr) if sr else '-'} | "
              f"{min(pubs) if pubs else '-'}..{max(pubs) if pubs else '-'} | {rel(pv[j])} | {kd} | {vd}")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "llama8b_64k"
    cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dev = torch.device("cuda:0")
    w = config_workload(name, seed=0)
    x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
    mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
    fwd = lambda: hta.hta_forward(*x, mask)  # noqa: E731
    if os.environ.get("FP8"):  # the forward over an E4M3 copy of the cache
        from workloads import fp8_cache
        k8, ks = fp8_cache(w.k_cache)
        v8, vs = fp8_cache(w.v_cache)
        k8, v8, ks, vs = k8.to(dev), v8.to(dev), ks.to(dev), vs.to(dev)
        fwd = lambda: hta.hta_forward_fp8kv(x[0], k8, v8, ks, vs, x[3], x[4], mask)  # noqa: E731
    if os.environ.get("PAGED"):  # the paged forward over in-order 16-key pages
        page = 16
        maxp = w.N // page
        kp = x[1].reshape(w.B * maxp, page, w.H_kv, w.d).contiguous()
        vp = x[2].reshape(w.B * maxp, page, w.H_kv, w.d).contiguous()
        bt = torch.arange(w.B * maxp, dtype=torch.int32, device=dev).view(w.B, maxp)
        fwd = lambda: hta.hta_forward_paged(x[0], kp, vp, bt, x[3], x[4], mask)  # noqa: E731
    L = hta.lib()
    t8 = bool(os.environ.get("T8"))  # the transposed FP8 kernel (prefix_t8.cu) instead
    if t8:
        L.hta_debug_set_trace = L.hta_debug_set_trace_t8
    L.hta_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = torch.zeros(32 * RECS, dtype=torch.int64, device=dev)
    fwd()
    torch.cuda.synchronize()
    assert L.hta_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), cta) == 0
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        buf.zero_()
        flush.zero_()
        flush.view(torch.float32).sum()
        fwd()
        torch.cuda.synchronize()
    L.hta_debug_set_trace(None, -1)
    raw = buf.cpu().view(32, RECS).tolist()
    ev = defaultdict(dict)  # (warp, event) -> {tile: clock}
    t0 = None
    for wi in range(32):
        last = 0
        hi = 0
        for r in raw[wi]:
            if r == 0:
                break
            r &= (1 << 64) - 1
            e, j, c = r >> 56, (r >> 32) & 0xFFFFFF, r & 0xFFFFFFFF
            c += hi
            if c < last:  # 32-bit wrap
                hi += 1 << 32
                c += 1 << 32
            last = c
            ev[(wi, e)][j] = c
            if e == 0:
                t0 = c if t0 is None else min(t0, c)
    if t0 is None:
        print("no trace records")
        return
    rel = lambda c: c - t0  # noqa: E731
    if t8:
        return analyze_t8(ev, rel, name, cta)
    exit_t = max(rel(v[0]) for (wi, e), v in ev.items() if e == 63)
    print(f"{name} CTA {cta}: exit at {exit_t} cycles after the first entry")
    # roles from the records: the MMA warp logs events 1-3, softmax warps event 10 (group = tile parity)
    mw = next((w for w in range(32) if (w, 1) in ev), 1)
    sm = [w for w in range(32) if (w, 10) in ev]
    grp = {w: min(ev[(w, 10)]) % 2 for w in sm}
    g0 = [w for w in sm if grp[w] == 0]
    g1 = [w for w in sm if grp[w] == 1]
    print(f"MMA warp {mw}; group 0 warps {g0}; group 1 warps {g1}")
    mma = {e: ev.get((mw, e), {}) for e in (1, 2, 3)}
    tiles = sorted(mma[1])
    if tiles:
        pv = [rel(mma[1][j]) for j in tiles]
        per = [b - a for a, b in zip(pv, pv[1:])]
        print(f"MMA: {len(tiles)} PV issues, first at {pv[0]}, last at {pv[-1]}; period median "
              f"{statistics.median(per) if per else 0:.0f} (p10 {sorted(per)[len(per) // 10] if per else 0}, "
              f"p90 {sorted(per)[9 * len(per) // 10] if per else 0})")
        # what gates PV_j: V landed (3) or P published (1 fires after 3)
        gate_v = [rel(mma[3][j]) for j in tiles if j in mma[3]]
        print(f"     V_j landed -> PV_j issued gap median {statistics.median([a - b for a, b in zip(pv, gate_v)]):.0f}")
        if mma[2]:
            s_is = [rel(mma[2][j]) for j in sorted(mma[2])]
            print(f"     S issues: first {s_is[0]}, K_0..2 landed at {s_is[:3]}")
    # FP8 cache producers: 30 -> 32 = K tile landed -> widened (warp of the K ring), 31 -> 33 (V)
    for a, b_, nm in ((30, 32, "K"), (31, 33, "V")):
        for wi in range(32):
            if (wi, b_) not in ev:
                continue
            st, en = ev[(wi, a)], ev[(wi, b_)]
            js = sorted(j for j in en if j in st)
            if not js:
                continue
            dur = [en[j] - st[j] for j in js]
            per = [en[y] - en[x] for x, y in zip(js, js[1:])]
            print(f"producer warp {wi} ({nm}): {len(js)} tiles widened; landed->widened median "
                  f"{statistics.median(dur):.0f}, widened period median {statistics.median(per) if per else 0:.0f}")
    for wi in sm:
        ten = ev.get((wi, 10), {})
        if not ten:
            continue
        rows = []
        for j in sorted(ten):
            r = [ev.get((wi, e), {}).get(j) for e in (10, 11, 12, 13, 15, 14)]
            if None in r:
                continue
            rows.append([r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4]])
        if not rows:
            continue
        med = [statistics.median(c[i] for c in rows) for i in range(5)]
        starts = sorted(ten)
        gaps = [ten[b] - ev[(wi, 14)][a] for a, b in zip(starts, starts[1:]) if a in ev[(wi, 14)]]
        print(f"softmax warp {wi:2d} (group {grp[wi]}): {len(rows)} tiles; median S ready->loaded "
              f"{med[0]:.0f}, exps {med[1]:.0f}, ->token {med[2]:.0f}, ->P stored {med[3]:.0f}, ->published {med[4]:.0f}; "
              f"idle waiting for S {statistics.median(gaps) if gaps else 0:.0f}")
    # timeline of a window of tiles: group warp 4 (even tiles) and 12 (odd tiles), MMA warp 1
    print("tile: S_j issued | S_j ready | loaded | exps done | token read | published | PV_j issued   (cycles)")
    mid = len(tiles) // 2 if tiles else 0
    for j in range(max(0, mid - 4), mid + 4):
        wi = g0[0] if j % 2 == 0 else g1[0]
        get = lambda w, e: ev.get((w, e), {}).get(j)  # noqa: E731
        vals = [get(mw, 2), get(wi, 10), get(wi, 11), get(wi, 12), get(wi, 13), get(wi, 14), get(mw, 1)]
        print(f"{j:4d}: " + " | ".join("-" if v is None else str(rel(v)) for v in vals))
    # critical chain per tile: S_j ready (first warp of its group) -> last warp of the group
    # published P_j -> PV_j issued -> S_{j+3} issued (by the MMA warp)
    print("tile: S ready(first) | P published (first..last warp) | PV_j issued | S_j+3 issued | S_j+3 ready")
    for j in range(max(0, mid - 6), mid + 6):
        ws = g0 if j % 2 == 0 else g1
        r10 = [ev.get((w, 10), {}).get(j) for w in ws]
        r14 = [ev.get((w, 14), {}).get(j) for w in ws]
        r10 = [rel(x) for x in r10 if x is not None]
        r14 = [rel(x) for x in r14 if x is not None]
        pv = ev.get((mw, 1), {}).get(j)
        s3 = ev.get((mw, 2), {}).get(j + 3)
        ws3 = g0 if (j + 3) % 2 == 0 else g1
        r3 = [ev.get((w, 10), {}).get(j + 3) for w in ws3]
        r3 = [rel(x) for x in r3 if x is not None]
        if r10 and r14:
            print(f"{j:4d}: {min(r10)} | {min(r14)}..{max(r14)} (+{max(r14) - min(r10)}) | "
                  f"{rel(pv) if pv else '-'} (+{rel(pv) - max(r14) if pv else 0}) | {rel(s3) if s3 else '-'} | "
                  f"{min(r3) if r3 else '-'} (+{min(r3) - rel(s3) if r3 and s3 else 0})")
    # producers: issue -> landed latency (V landed = event 3 of the MMA warp, K landed = event 2)
    kw = next((w for w in range(32) if (w, 30) in ev), None)
    vw = next((w for w in range(32) if (w, 31) in ev), None)
    if kw is not None and vw is not None and (kw, 32) not in ev and not any((w, 34) in ev for w in range(32)):
        kl = [mma[2][j] - ev[(kw, 30)][j] for j in tiles if j in mma[2] and j in ev[(kw, 30)]]
        vl = [mma[3][j] - ev[(vw, 31)][j] for j in tiles if j in mma[3] and j in ev[(vw, 31)]]
        vlead = [mma[1][j] - ev[(vw, 31)][j] for j in tiles if j in ev[(vw, 31)]]
        print(f"producers: K issue->landed(+S issue) median {statistics.median(kl):.0f}, V issue->landed median "
              f"{statistics.median(vl):.0f}, V issue -> PV_j issue median {statistics.median(vlead):.0f}")
    # FP8 cache: per producer, landed (30/31) -> widened (32/33) and the gap between tiles
    for e0, e1, nm in ((30, 32, "K"), (31, 33, "V")):
        w0 = next((w for w in range(32) if (w, e1) in ev), None)
        if w0 is None:
            continue
        a, bb = ev[(w0, e0)], ev[(w0, e1)]
        js = sorted(j for j in bb if j in a)
        if len(js) < 2:
            continue
        wid = [bb[j] - a[j] for j in js]
        gap = [a[j2] - bb[j1] for j1, j2 in zip(js, js[1:])]
        print(f"FP8 {nm} producer (warp {w0}): widen median {statistics.median(wid):.0f} cycles, "
              f"wait for the next tile to land median {statistics.median(gap):.0f}")
    # FP8 cache, widening warps (<= 64 rows): landed (34) -> widened (32 K / 33 V), and the wait
    # for the next tile to land
    for wi in range(32):
        if (wi, 34) not in ev:
            continue
        e1 = 32 if (wi, 32) in ev else 33
        a, bb = ev[(wi, 34)], ev.get((wi, e1), {})
        js = sorted(j for j in bb if j in a)
        if not js:
            continue
        wid = [bb[j] - a[j] for j in js]
        gap = [a[j2] - bb[j1] for j1, j2 in zip(js, js[1:])]
        c35 = ev.get((wi, 35), {})
        fen = [bb[j] - c35[j] for j in js if j in c35]
        print(f"widening warp {wi} ({'K' if e1 == 32 else 'V'}): widen median {statistics.median(wid):.0f} "
              f"(fence + sync {statistics.median(fen) if fen else 0:.0f}), "
              f"wait for the next landing median {statistics.median(gap) if gap else 0:.0f}, "
              f"widened at {[rel(bb[j]) for j in js[:4]]}..")
    # per warp: median lag of its publish behind the first warp of its group
    lags = defaultdict(list)
    for j in range(2, len(tiles) - 2):
        ws = list(g0 if j % 2 == 0 else g1)
        t = {w: ev.get((w, 14), {}).get(j) for w in ws}
        if None in t.values():
            continue
        t0 = min(t.values())
        for w in ws:
            lags[w].append(t[w] - t0)
    print("publish lag behind the group's first warp (median):",
          {w: int(statistics.median(v)) for w, v in sorted(lags.items())})
    if "--raw" in sys.argv:
        for (wi, e), v in sorted(ev.items()):
            print(wi, e, [(j, rel(c)) for j, c in sorted(v.items())][:12])


if __name__ == "__main__":
    main()
