"""CPU tests of the C ABI: the library loads, exports every symbol include/hta.h declares, and
its host-side logic (workspace sizing, argument validation, host tree utilities) is right.
No compute call is made (no GPU here)."""
import ctypes
import itertools
import os
import re

import numpy as np
import pytest
import torch

import oracle
from workloads import accept_tokens, tree_parents
from paper_2502_17421_b200 import hta

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2502_17421_b200 import build
    build.build()
    return hta.lib()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "hta.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hta_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_header_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(hta._SIG), "binding and header disagree"


def test_status_strings_and_version(L):
    for code, name in hta.STATUS.items():
        assert L.hta_status_string(code).decode() == name
    assert L.hta_version() >= 100


def _shape(B=1, T=64, H=32, H_kv=8, d=128, N=65536, dtype=hta.HTA_BF16, splits=0):
    s = hta.hta_shape_t()
    s.B, s.T, s.H, s.H_kv, s.d, s.N_max = B, T, H, H_kv, d, N
    s.softmax_scale = 1.0 / d ** 0.5
    s.dtype = dtype
    s.num_splits = splits
    return s


def test_workspace_size_matches_split_plan(L):
    part = lambda s: (s.B * s.T * s.H * s.d + s.B * s.H * s.T) * 4
    # Llama-8B-64k: M = 256 rows per kv head -> one CTA pair per kv head, 8 pairs = 16 CTAs per
    # split, 9 splits = 144 CTAs
    s = _shape()
    assert L.hta_workspace_size(ctypes.byref(s), 148) == 9 * part(s)
    # forced splits are capped by the number of 128-key tiles (and rounded to whole tiles per
    # split); the size covers the larger of the plans without and with the fused tree pass's
    # tree tile (hta_forward): N=300: 3 tiles -> 3 splits, 3 + 1 tree tile -> 4 splits;
    # N=1000: 8 tiles in 7 splits = 2 per split = 4 splits, 8 + 1 -> 2 per split = 5 splits
    s = _shape(N=300, splits=7)
    assert L.hta_workspace_size(ctypes.byref(s), 148) == 4 * part(s)
    s = _shape(N=1000, splits=7)
    assert L.hta_workspace_size(ctypes.byref(s), 148) == 5 * part(s)
    s = _shape(N=0)
    assert L.hta_workspace_size(ctypes.byref(s), 148) == 1 * part(s)
    # QwQ-like: M = 320 rows.  Pairs: 2 row groups x 8 kv heads x B=4 = 128 CTAs per split, best
    # 1 split (one wave of 256 tiles).  Single CTAs: 3 row groups = 96 CTAs per split, 3 splits =
    # 288 CTAs = 2 waves of 86 tiles -> the planner takes single CTAs with 3 splits
    s = _shape(B=4, H=40, N=32768)
    assert L.hta_workspace_size(ctypes.byref(s), 148) == 3 * part(s)


@pytest.mark.parametrize("field,value", [("T", 0), ("T", 257), ("H", 30), ("d", 96), ("N_max", -1),
                                         ("softmax_scale", 0.0), ("softmax_scale", float("nan")),
                                         ("max_seqlen", -1), ("num_splits", -2), ("dtype", 7)])
def test_invalid_shapes_rejected_on_host(L, field, value):
    s = _shape()
    setattr(s, field, value)
    assert L.hta_workspace_size(ctypes.byref(s), 148) == ctypes.c_size_t(-1).value
    # the compute entry points reject it before touching the device
    rc = L.hta_forward(ctypes.byref(s), *([ctypes.c_void_p(16)] * 7), 0, ctypes.c_void_p(16), None,
                       ctypes.c_void_p(16), 1 << 30, None)
    assert rc in (1, 2)


def test_misaligned_strides_rejected(L):
    s = _shape()
    s.q_strides = (ctypes.c_int64 * 3)(64 * 32 * 128, 32 * 128, 127)
    assert L.hta_workspace_size(ctypes.byref(s), 148) == ctypes.c_size_t(-1).value


def test_null_pointers_rejected(L):
    s = _shape(N=256)
    rc = L.hta_forward(ctypes.byref(s), None, *([ctypes.c_void_p(16)] * 6), 0, ctypes.c_void_p(16), None,
                       ctypes.c_void_p(16), 1 << 30, None)
    assert rc == 1


def test_host_mask_builder_bit_exact_vs_oracle(L):
    for seed in range(40):
        T = [1, 2, 8, 17, 64, 128, 200, 256][seed % 8]
        kind = ["random", "random_forest", "beam", "chain", "star", "heap_binary", "roots"][seed % 7]
        par = tree_parents(kind, T, seed=seed)
        m = hta.hta_build_tree_mask(par)
        np.testing.assert_array_equal(m.numpy(), oracle.tree_mask(par))
        assert hta.hta_validate_tree_mask(m)


def test_host_mask_builder_rejects_bad_parents(L):
    for bad in ([0], [-1, 1], [-1, 0, 3], [-3, -1]):
        with pytest.raises(hta.HtaError):
            hta.hta_build_tree_mask(torch.tensor(bad, dtype=torch.int32))


def test_validator_rejects_non_tree_masks(L):
    good = oracle.tree_mask(tree_parents("heap_binary", 8))
    assert hta.hta_validate_tree_mask(torch.from_numpy(good))
    bad = good.copy()
    bad[3, 3] = 0                       # not reflexive
    assert not hta.hta_validate_tree_mask(torch.from_numpy(bad))
    bad = good.copy()
    bad[1, 5] = 1                       # sees a later node
    assert not hta.hta_validate_tree_mask(torch.from_numpy(bad))
    bad = good.copy()
    bad[7, 0] = 0                       # not ancestor-closed (misses the root)
    assert not hta.hta_validate_tree_mask(torch.from_numpy(bad))


def test_host_accept_bit_exact_vs_oracle(L):
    for seed in range(400):
        T = [1, 3, 8, 17, 64, 128, 256][seed % 7]
        kind = ["random", "random_forest", "beam", "chain", "star"][seed % 5]
        par = tree_parents(kind, T, seed=seed)
        draft, tgt, ctx = accept_tokens(par, seed, vocab=4, p_match=0.8, distinct_siblings=(seed % 2 == 0))
        for root in (0, -1) if kind != "random_forest" else (-1,):
            got = hta.hta_accept_greedy(par, draft, tgt, root=root, context_argmax=ctx)
            want = oracle.accept_greedy(par, draft, tgt, root=root, context_argmax=ctx)
            assert got == (want[0], want[1]), (seed, root)


def test_host_accept_exhaustive_small(L):
    for T in range(1, 5):
        for par in itertools.product(*[range(-1, i) for i in range(T)]):
            p = torch.tensor(par, dtype=torch.int32)
            for bits in range(1 << T):
                draft = torch.tensor([(bits >> i) & 1 for i in range(T)], dtype=torch.int32)
                tgt = torch.tensor([(bits >> ((i + 1) % T)) & 1 for i in range(T)], dtype=torch.int32)
                for root in range(-1, T):
                    got = hta.hta_accept_greedy(p, draft, tgt, root=root, context_argmax=1)
                    want = oracle.accept_greedy(par, draft, tgt, root=root, context_argmax=1)
                    assert got == (want[0], want[1])


def test_shard_bounds_cover_sequence():
    for N in (0, 1, 7, 65536, 131071):
        for P in (1, 2, 3, 4, 8):
            b = [hta.shard_bounds(N, P, r) for r in range(P)]
            assert b[0][0] == 0 and b[-1][1] == N
            assert all(b[i][1] == b[i + 1][0] for i in range(P - 1))
            assert max(hi - lo for lo, hi in b) - min(hi - lo for lo, hi in b) <= 1


def test_loopback_communicator_host_checks(L):
    """Loopback communicator (P virtual ranks, no NCCL): host-side creation and argument checks."""
    h = ctypes.c_void_p()
    assert L.hta_comm_create_loopback(0, ctypes.byref(h)) == 1
    assert L.hta_comm_create_loopback(65, ctypes.byref(h)) == 1
    assert L.hta_comm_create_loopback(4, ctypes.byref(h)) == 0
    try:
        assert L.hta_comm_async_error(h) == 0
        s = _shape(N=2048)
        # a loopback communicator is not an NCCL one: hta_forward_seqpar refuses it
        rc = L.hta_forward_seqpar(h, ctypes.byref(s), *([ctypes.c_void_p(16)] * 7), 0, ctypes.c_void_p(16), None,
                                  0, ctypes.c_void_p(16), 1 << 30, None)
        assert rc == 1
        # NULL per-rank pointer arrays are rejected before any device work
        rc = L.hta_forward_seqpar_loopback(h, ctypes.byref(s), ctypes.c_void_p(16), None, None, None,
                                           ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16), 0, None,
                                           None, 0, ctypes.c_void_p(16), 1 << 30, None)
        assert rc == 1
        # H not divisible by the rank count
        s = _shape(H=12, H_kv=4, N=2048)
        assert L.hta_workspace_size_seqpar(ctypes.byref(s), 148, 8) == ctypes.c_size_t(-1).value
    finally:
        assert L.hta_comm_destroy(h) == 0


def test_seqpar_workspace_layout(L):
    """hta_workspace_size_seqpar = split partials + send and receive blocks [P][blk] + own output
    slice + the gathered slices (16-byte rounded pieces)."""
    r16 = lambda x: (x + 15) // 16 * 16
    for P, B, T in ((1, 1, 64), (2, 1, 64), (4, 1, 64), (8, 1, 64), (8, 2, 13)):
        s = _shape(B=B, T=T, N=16384)
        blk = (s.B * s.T * (s.H // P) * s.d + s.B * (s.H // P) * s.T + 3) // 4 * 16
        o_sl = s.B * s.T * (s.H // P) * s.d * 2
        l_sl = s.B * (s.H // P) * s.T * 4
        want = r16(L.hta_workspace_size(ctypes.byref(s), 148)) + 2 * r16(P * blk) + r16(o_sl) + r16(l_sl) + \
            r16(P * o_sl) + r16(P * l_sl)
        assert L.hta_workspace_size_seqpar(ctypes.byref(s), 148, P) == want


def test_max_seqlen_hint_shrinks_the_plan(L):
    """With a 128k-capacity cache filled to 8k, the hint plans 8k keys: fewer tiles, so the split
    count (and workspace) is that of an 8k cache, not of the capacity."""
    part = lambda s: (s.B * s.T * s.H * s.d + s.B * s.H * s.T) * 4
    full = _shape(N=131072)
    hinted = _shape(N=131072)
    hinted.max_seqlen = 8192
    small = _shape(N=8192)
    assert L.hta_workspace_size(ctypes.byref(hinted), 148) == L.hta_workspace_size(ctypes.byref(small), 148)
    assert L.hta_workspace_size(ctypes.byref(full), 148) >= L.hta_workspace_size(ctypes.byref(hinted), 148)
    assert L.hta_workspace_size(ctypes.byref(hinted), 148) % part(hinted) == 0
