"""CPU fp64 oracle for Hybrid Tree Attention -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and bench.py's `cpu_baseline` / `--impl reference`
legs may import this package.  The product library (`paper_2502_17421_b200`) never imports
it and shares no code with it; see DESIGN.md "Oracle".

Contents
  attention(...)     explicit-mask fp64 attention (C, hta_oracle.c), steps O1-O7 of
                     SURVEY.md §8(c) / PAPER.md:195-201, 603-656.
  merge(parts)       the LSE aggregation of PAPER.md:203-219 (max-shifted, reading Z11).
  tree_mask(...)     ancestor mask by recursive set walk (oracle/tree.py).
  accept_greedy(...) longest accepted root path by brute-force enumeration (oracle/tree.py).
  commit_kv(...)     append the accepted nodes' K/V rows to the cache in path order (oracle/tree.py).
  attention_fp8kv(...) attention over an FP8 (E4M3) cache decoded from its definition (oracle/fp8.py).

Parity status of each function is recorded in DESIGN.md "Oracle pins".
"""
from .attention import attention, merge, load_library, build_library  # noqa: F401
from .tree import tree_mask, accept_greedy, commit_kv  # noqa: F401
from .fp8 import attention_fp8kv, decode_e4m3, e4m3_value  # noqa: F401
