"""Negative controls (SURVEY.md §4 "a --sabotage merge mode must fail parity", in the spirit of
S:581): the parity check used everywhere (gpu_util.compare, the north_star tolerances) must
REJECT a forward whose merge or mask has a plausible bug.  Each sabotage re-runs the three ABI
steps (hta_prefix_attn, hta_tree_attn, hta_merge_lse) on the GPU with one input corrupted the way
a merge/mask bug would corrupt it, and asserts that the comparison with the oracle fails, while
the unsabotaged composition passes."""
import numpy as np
import pytest
import torch

import oracle
from paper_2502_17421_b200 import hta
from workloads import make_workload

from gpu_util import compare, oracle_masks

pytestmark = pytest.mark.gpu

SABOTAGES = ["none", "drop_tree_part", "tree_lse_plus_ln2", "prefix_lse_minus_ln2", "swap_parts_lse",
             "transposed_mask", "self_only_mask", "drop_cache_split"]


@pytest.fixture(scope="module")
def case(cuda_device):
    w = make_workload(1, 64, 32, 8, 128, 4000, "bf16", dist="V1", seed=7, tree="beam")
    mask = oracle_masks(w)
    o_ref, l_ref = oracle.attention(w.q, w.k_cache, w.v_cache, w.k_tree, w.v_tree, mask)
    x = {k: getattr(w, k).to(cuda_device) for k in ("q", "k_cache", "v_cache", "k_tree", "v_tree")}
    return w, mask, o_ref, l_ref, x


def _composed(x, mask_np, sabotage, dev):
    m = mask_np[0]
    if sabotage == "transposed_mask":
        m = m.T.copy()
    elif sabotage == "self_only_mask":
        m = np.eye(m.shape[0], dtype=np.uint8)
    mask = torch.from_numpy(np.ascontiguousarray(m)).to(dev)
    if sabotage == "drop_cache_split":
        # a dropped split-KV part: the prefix pass over only the first half of the cache
        n = x["k_cache"].shape[1] // 2
        o_c, l_c = hta.hta_prefix_attn(x["q"], x["k_cache"][:, :n].contiguous(), x["v_cache"][:, :n].contiguous())
    else:
        o_c, l_c = hta.hta_prefix_attn(x["q"], x["k_cache"], x["v_cache"])
    o_s, l_s = hta.hta_tree_attn(x["q"], x["k_tree"], x["v_tree"], mask)
    if sabotage == "tree_lse_plus_ln2":
        l_s = l_s + float(np.log(2.0))
    elif sabotage == "prefix_lse_minus_ln2":
        l_c = l_c - float(np.log(2.0))
    elif sabotage == "swap_parts_lse":
        l_c, l_s = l_s, l_c
    if sabotage == "drop_tree_part":
        parts_o, parts_l = o_c[None], l_c[None]
    else:
        parts_o, parts_l = torch.stack([o_c, o_s]), torch.stack([l_c, l_s])
    o, lse = hta.hta_merge_lse(parts_o, parts_l, dtype=torch.bfloat16, H_kv=x["k_cache"].shape[2])
    torch.cuda.synchronize()
    return o, lse


@pytest.mark.parametrize("sabotage", SABOTAGES)
def test_sabotaged_merge_fails_parity(cuda_device, case, sabotage):
    w, mask, o_ref, l_ref, x = case
    o, lse = _composed(x, mask, sabotage, cuda_device)
    if sabotage == "none":
        compare(o, lse, o_ref, l_ref, "bf16", "unsabotaged composition")
    else:
        with pytest.raises(AssertionError):
            compare(o, lse, o_ref, l_ref, "bf16", f"sabotage {sabotage}")
        # the O tolerances alone (max 2e-2, mean 2e-3) catch it too, not only the LSE bound
        with pytest.raises(AssertionError):
            compare(o, None, o_ref, l_ref, "bf16", f"sabotage {sabotage} (O only)")
