import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_2502_17421_b200 import hta
from workloads.generators import named_generator
dev = torch.device('cuda:0')
for key, d in [(434, 64), (434, 128), (3, 64), (194, 64)]:
    B, T, H, Hkv, N = 1, 4, 4, 1, 576
    gen = named_generator(11, f"jump:{key}:{d}")
    u = torch.randn(d, generator=gen); u = u / u.norm()
    tdt = torch.bfloat16
    q = (40.0 * u + 0.5 * torch.randn(B, T, H, d, generator=gen)).to(tdt)
    kc = torch.randn(B, N, Hkv, d, generator=gen)
    kc[:, key, :, :] = 42.5 * u + 0.1 * kc[:, key, :, :]
    kc = kc.to(tdt)
    vc = torch.randn(B, N, Hkv, d, generator=gen).to(tdt)
    kt = torch.zeros(B, T, Hkv, d, dtype=tdt)
    mask = np.ones((B, T, T), np.uint8)
    oc_ref, lc_ref = oracle.attention(q, kc, vc, kt, kt, mask, part="cache")
    oc, lc = hta.hta_prefix_attn(q.to(dev), kc.to(dev), vc.to(dev), num_splits=1)
    torch.cuda.synchronize()
    e = np.abs(oc.cpu().numpy() - oc_ref)
    print(key, d, "row max err", np.round(e.reshape(-1, d).max(1), 4), "lse", np.round(lc.cpu().numpy().ravel() - lc_ref.ravel(), 4))
