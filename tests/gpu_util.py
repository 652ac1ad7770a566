"""Shared helpers of the GPU parity tests: run a workload through libhta and the oracle."""
import numpy as np
import torch

import oracle

# BASELINE.json north_star tolerances.
BF16_MAX_ABS = 2e-2
BF16_MEAN_ABS = 2e-3
BF16_LSE_ABS = 1e-3    # reading Z16 (LSE of bf16 inputs with fp32 accumulation)
FP32_REL = 1e-5        # reading Z15 (per-row relative)


def oracle_masks(w):
    return np.stack([oracle.tree_mask(w.parents[b]) for b in range(w.B)]) if w.T > 0 else \
        np.zeros((w.B, 0, 0), np.uint8)


def to_dev(w, dev):
    return dict(q=w.q.to(dev), kc=w.k_cache.to(dev), vc=w.v_cache.to(dev), kt=w.k_tree.to(dev),
                vt=w.v_tree.to(dev), sl=w.seqlens.to(dev))


def compare(o_gpu, lse_gpu, o_ref, lse_ref, dtype, what=""):
    """Assert the north_star tolerances.  o_* [B,T,H,d] (or [R,d]); lse_* [B,H,T] (or [R])."""
    o = o_gpu.float().cpu().numpy().astype(np.float64)
    ref = np.asarray(o_ref, np.float64)
    lg = None if lse_gpu is None else lse_gpu.float().cpu().numpy().astype(np.float64)
    lr = np.asarray(lse_ref, np.float64)
    # sentinels must match exactly (O = 0, LSE = -inf) and nothing may be NaN
    assert not np.isnan(o).any(), f"{what}: NaN in O"
    if lg is not None:
        assert not np.isnan(lg).any(), f"{what}: NaN in LSE"
        np.testing.assert_array_equal(np.isneginf(lg), np.isneginf(lr), err_msg=f"{what}: sentinel rows differ")
        fin = np.isfinite(lr)
    err = np.abs(o - ref)
    stats = dict(max_abs=float(err.max(initial=0)), mean_abs=float(err.mean()) if err.size else 0.0)
    if dtype == "bf16":
        assert stats["max_abs"] <= BF16_MAX_ABS, f"{what}: max abs {stats}"
        assert stats["mean_abs"] <= BF16_MEAN_ABS, f"{what}: mean abs {stats}"
        if lg is not None and fin.any():
            le = np.abs(lg[fin] - lr[fin]).max()
            stats["lse_max_abs"] = float(le)
            assert le <= BF16_LSE_ABS, f"{what}: lse {le}"
    else:
        rows_o = o.reshape(-1, o.shape[-1])
        rows_r = ref.reshape(-1, ref.shape[-1])
        rel = np.abs(rows_o - rows_r).max(axis=1) / np.maximum(np.abs(rows_r).max(axis=1), 1e-6)
        stats["row_rel_max"] = float(rel.max(initial=0))
        assert stats["row_rel_max"] <= FP32_REL, f"{what}: fp32 row rel {stats}"
        if lg is not None and fin.any():
            le = (np.abs(lg[fin] - lr[fin]) / np.maximum(1.0, np.abs(lr[fin]))).max()
            stats["lse_rel_max"] = float(le)
            assert le <= FP32_REL, f"{what}: fp32 lse {le}"
    return stats
