"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no attention, no masks built from trees,
no softmax, no merge).  It only draws random tensors and random parent arrays, so that
the oracle (`oracle/`) and the CUDA path (`paper_2502_17421_b200/`) can be fed identical
inputs without either importing the other.  See DESIGN.md "Input recipe".
"""
from .generators import (  # noqa: F401
    BASE_SEED,
    CONFIGS,
    Workload,
    make_workload,
    named_generator,
    tree_parents,
    beam_tree,
    random_mask,
    accept_tokens,
    fp8_cache,
)
