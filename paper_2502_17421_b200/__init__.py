"""B200-native Hybrid Tree Attention (LongSpec, arXiv 2502.17421).

The computation lives in libhta.so (CUDA, sm_100a; C ABI in include/hta.h).  This package is
its thin Python binding; see DESIGN.md for the design and README.md for usage.
"""
from .hta import (  # noqa: F401
    HtaComm,
    HtaError,
    hta_accept_greedy,
    hta_build_tree_mask,
    hta_forward,
    hta_merge_lse,
    hta_prefix_attn,
    hta_tree_attn,
    hta_validate_tree_mask,
    lib,
    make_shape,
    shard_bounds,
    workspace_size,
)
