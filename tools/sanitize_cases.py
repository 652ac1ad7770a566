"""Small invocations of every kernel family for compute-sanitizer (diagnostics; tools/, not the
product).  Each case runs once and is checked against the oracle, so a tool that perturbs the
kernels (racecheck / initcheck / synccheck serialise them) still has to reproduce the result.

    compute-sanitizer --tool {memcheck|racecheck|initcheck|synccheck} python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from gpu_util import compare, oracle_masks, to_dev  # noqa: E402
from paper_2502_17421_b200 import hta  # noqa: E402
from workloads import fp8_cache, make_workload  # noqa: E402

CASES = [
    # B, T, H, Hkv, d, N, dtype, tree: toy fp32, CTA pair, MHA single CTA (fused tree), G = 5, d = 64
    (1, 8, 1, 1, 64, 256, "fp32", "heap_binary"),
    (1, 64, 32, 8, 128, 1000, "bf16", "beam"),
    (1, 64, 4, 4, 128, 700, "bf16", "beam"),
    (2, 30, 10, 2, 128, 500, "bf16", "random"),
    (1, 17, 4, 1, 64, 300, "bf16", "star"),
]


def main():
    dev = torch.device("cuda:0")
    for B, T, H, Hkv, d, N, dt, tree in CASES:
        w = make_workload(B, T, H, Hkv, d, N, dt, dist="V1", seed=3, tree=tree)
        x = to_dev(w, dev)
        masks = oracle_masks(w)
        o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, masks)
        mask = torch.from_numpy(masks).to(dev)  # [B, T, T] (the trees of a batch may differ)
        o, l = hta.hta_forward(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], mask)
        torch.cuda.synchronize()
        compare(o, l, o_ref, l_ref, dt, f"forward {B, T, H, Hkv, d, N, dt}")
        if dt == "bf16":
            par = torch.stack([w.parents[b] for b in range(B)]).to(torch.int32).to(dev)
            o2, l2 = hta.hta_forward_tree(x["q"], x["kc"], x["vc"], x["kt"], x["vt"], par)
            torch.cuda.synchronize()
            assert torch.equal(o, o2) and torch.equal(l, l2)
            k8, ks = fp8_cache(w.k_cache)
            v8, vs = fp8_cache(w.v_cache)
            o8_ref, l8_ref = oracle.attention_fp8kv(w.q, k8, v8, ks, vs, w.k_tree, w.v_tree, masks)
            o8, l8 = hta.hta_forward_fp8kv(x["q"], k8.to(dev), v8.to(dev), ks.to(dev), vs.to(dev), x["kt"], x["vt"],
                                           mask)
            torch.cuda.synchronize()
            compare(o8, l8, o8_ref, l8_ref, "bf16", "fp8 forward")
        print(f"ok {B, T, H, Hkv, d, N, dt, tree}", flush=True)
    # tree step (a0 + a6) and the paged forward
    par = make_workload(1, 64, 8, 2, 128, 512, "bf16", seed=4, tree="beam").parents[0].to(dev)
    m = hta.hta_build_tree_mask(par)
    assert np.array_equal(m.cpu().numpy(), oracle.tree_mask(par.cpu()))
    w = make_workload(1, 64, 8, 2, 128, 512, "bf16", dist="V1", seed=5, tree="beam")
    x = to_dev(w, dev)
    kp = x["kc"].reshape(32, 16, 2, 128).contiguous()
    vp = x["vc"].reshape(32, 16, 2, 128).contiguous()
    bt = torch.arange(32, dtype=torch.int32, device=dev).flip(0).view(1, 32).contiguous()
    kp, vp = kp.flip(0).contiguous(), vp.flip(0).contiguous()
    masks = oracle_masks(w)
    o, l = hta.hta_forward_paged(x["q"], kp, vp, bt, x["kt"], x["vt"], torch.from_numpy(masks).to(dev))
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, masks)
    torch.cuda.synchronize()
    compare(o, l, o_ref, l_ref, "bf16", "paged")
    print("ok tree step, paged", flush=True)


if __name__ == "__main__":
    main()
