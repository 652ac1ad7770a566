"""Pipeline timeline of one CTA of the two-Q-tile prefix variant (tools/variants_src/prefix_q2.inc, built with -DHTA_TRACE).

    HTA_LIB=... WPG=8 python tools/trace_q2.py [cta]
"""
import ctypes, os, sys, statistics
ROOT = "/root/repo"; sys.path.insert(0, ROOT)
import torch
from paper_2502_17421_b200 import hta
from workloads.generators import config_workload
dev = torch.device("cuda:0")
w = config_workload("llama8b_64k", seed=0)
x = [t.to(dev) for t in (w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree)]
mask = hta.hta_build_tree_mask(w.parents[0].to(dev))
L = hta.lib()
L.hta_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = torch.zeros(32 * 2048, dtype=torch.int64, device=dev)
hta.hta_forward(*x, mask); torch.cuda.synchronize()
assert L.hta_debug_set_trace(ctypes.c_void_p(buf.data_ptr()), int(sys.argv[1]) if len(sys.argv) > 1 else 0) == 0
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    buf.zero_(); flush.zero_(); hta.hta_forward(*x, mask); torch.cuda.synchronize()
ev = {}
for warp, row in enumerate(buf.view(32, 2048).cpu().tolist()):
    for v in row:
        if v == 0: break
        v &= (1 << 64) - 1
        e, tag, j, c = v >> 56, (v >> 52) & 0xF, (v >> 32) & 0xFFFFF, v & 0xFFFFFFFF
        if e < 50: ev[(e, tag, j)] = c
t0 = min(ev.values())
ev = {k: v - t0 for k, v in ev.items()}
js = sorted({k[2] for k in ev})
WPG = int(os.environ.get("WPG", "8"))
print("  j | g | S iss  S rdy  ld  exp  pub(max)  Pseen | period")
prev = {}
for j in js:
    for g in (0, 1):
        ws = range(WPG * g, WPG * g + WPG)
        g_ = lambda e, t: ev.get((e, t, j), -1)
        rdy = min([g_(10, t) for t in ws if g_(10, t) >= 0] or [-1])
        rdy_max = max([g_(10, t) for t in ws] or [-1])
        ld = max([g_(11, t) for t in ws] or [-1]); ex = max([g_(12, t) for t in ws] or [-1]); pub = max([g_(13, t) for t in ws] or [-1])
        per = rdy - prev.get(g, rdy); prev[g] = rdy
        print(f"{j:3d} | {g} | {g_(21, g):6d} {rdy:6d} {ld-rdy:4d} {ex-ld:4d} {pub-ex:4d} {pub:8d} {g_(1, g)-pub:5d} | {per}  (S seen spread {rdy_max-rdy})")
jm = js[len(js) // 2]
print(f"tile {jm}, per softmax warp: S seen, +ld, +exp, +pub (cycles)")
for t in range(2 * WPG):
    a = [ev.get((e, t, jm), -1) for e in (10, 11, 12, 13)]
    print(f"  warp {t + 2:2d} (group {t // WPG}): {a[0]:8d} {a[1]-a[0]:5d} {a[2]-a[1]:5d} {a[3]-a[2]:5d}")
