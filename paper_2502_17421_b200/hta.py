"""ctypes binding of libhta (include/hta.h).  Argument marshalling only.

Every function here packs torch tensors into the C ABI's pointers/shape struct and calls the
library; all computation runs in libhta's CUDA kernels (or, for the `on_device=0` tree
utilities, in libhta's host code).  There is no fallback: if libhta.so is missing or the device
is not sm_100 the calls raise.  PyTorch provides device memory and the current stream only.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HTA_LIB", os.path.join(_PKG, "libhta.so"))

HTA_BF16, HTA_FP32 = 0, 1
STATUS = {0: "HTA_OK", 1: "HTA_ERR_INVALID_ARGUMENT", 2: "HTA_ERR_UNSUPPORTED", 3: "HTA_ERR_INVALID_MASK",
          4: "HTA_ERR_WORKSPACE", 5: "HTA_ERR_CUDA", 6: "HTA_ERR_NCCL"}


class HtaError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)}")
        self.code = code


class hta_shape_t(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("T", ctypes.c_int32), ("H", ctypes.c_int32), ("H_kv", ctypes.c_int32),
                ("d", ctypes.c_int32), ("N_max", ctypes.c_int64), ("softmax_scale", ctypes.c_float),
                ("dtype", ctypes.c_int32), ("q_strides", ctypes.c_int64 * 3), ("kv_strides", ctypes.c_int64 * 3),
                ("tkv_strides", ctypes.c_int64 * 3), ("num_splits", ctypes.c_int32), ("max_seqlen", ctypes.c_int32)]


_lib = None
_P = ctypes.c_void_p
_SIG = {
    "hta_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "hta_version": (ctypes.c_int32, []),
    "hta_workspace_size": (ctypes.c_size_t, [ctypes.POINTER(hta_shape_t), ctypes.c_int32]),
    "hta_prefix_attn": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P]),
    "hta_tree_attn": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, ctypes.c_int64, _P, _P, _P]),
    "hta_merge_lse": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), ctypes.c_int32, _P, _P, _P, _P, _P]),
    "hta_forward": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P, ctypes.c_int64, _P, _P,
                                   _P, ctypes.c_size_t, _P]),
    "hta_forward_timed": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P, ctypes.c_int64,
                                         _P, _P, _P, ctypes.c_size_t, _P, _P, _P]),
    "hta_forward_ex": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P, ctypes.c_int64, _P, _P,
                                      _P, ctypes.c_size_t, _P, _P]),
    "hta_forward_tree": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P, ctypes.c_int64,
                                        _P, _P, _P, ctypes.c_size_t, _P, _P, _P, _P]),
    "hta_forward_paged": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, ctypes.c_int32, ctypes.c_int32, _P,
                                         ctypes.c_int32, _P, _P, _P, _P, ctypes.c_int64, _P, _P, _P, ctypes.c_size_t,
                                         _P]),
    "hta_forward_fp8kv": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                         ctypes.c_int64, _P, _P, _P, ctypes.c_size_t, _P]),
    "hta_prefix_attn_fp8kv": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                             ctypes.c_size_t, _P]),
    "hta_build_tree_mask": (ctypes.c_int, [_P, ctypes.c_int32, _P, ctypes.c_int32, _P]),
    "hta_validate_tree_mask": (ctypes.c_int, [_P, ctypes.c_int32]),
    "hta_accept_greedy": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P,
                                         ctypes.c_int32, _P]),
    "hta_tree_step": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P, _P, ctypes.c_int32, ctypes.c_int32, _P, _P, _P, _P]),
    "hta_commit_kv": (ctypes.c_int, [ctypes.POINTER(hta_shape_t), _P, ctypes.c_int64, _P, _P, _P, _P, _P, _P, _P, _P]),
    "hta_comm_unique_id": (ctypes.c_int, [_P]),
    "hta_comm_create": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "hta_comm_destroy": (ctypes.c_int, [_P]),
    "hta_comm_create_loopback": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "hta_comm_async_error": (ctypes.c_int, [_P]),
    "hta_comm_p2p_alloc": (ctypes.c_int, [_P, ctypes.c_size_t, _P]),
    "hta_comm_p2p_open": (ctypes.c_int, [_P, _P]),
    "hta_comm_p2p_set": (ctypes.c_int, [_P, ctypes.c_int32]),
    "hta_comm_p2p_error": (ctypes.c_int, [_P]),
    "hta_workspace_size_seqpar": (ctypes.c_size_t, [ctypes.POINTER(hta_shape_t), ctypes.c_int32, ctypes.c_int32]),
    "hta_forward_seqpar": (ctypes.c_int, [_P, ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P,
                                          ctypes.c_int64, _P, _P, ctypes.c_int32, _P, ctypes.c_size_t, _P]),
    "hta_forward_seqpar_tree": (ctypes.c_int, [_P, ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P,
                                               ctypes.c_int64, _P, _P, ctypes.c_int32, _P, ctypes.c_size_t, _P]),
    "hta_forward_seqpar_loopback": (ctypes.c_int, [_P, ctypes.POINTER(hta_shape_t), _P, _P, _P, _P, _P, _P, _P,
                                                   ctypes.c_int64, _P, _P, ctypes.c_int32, _P, ctypes.c_size_t,
                                                   _P]),
}


def lib():
    """Load libhta.so (raises if it has not been built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libhta.so not found at {LIB_PATH}; run `python -m paper_2502_17421_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(fn: str, code: int):
    if code != 0:
        raise HtaError(fn, code)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return HTA_BF16
    if dt == torch.float32:
        return HTA_FP32
    raise TypeError(f"unsupported dtype {dt}")


def _strides3(t: torch.Tensor):
    if t.stride(-1) != 1:
        raise ValueError("innermost (head-dim) stride must be 1")
    return (ctypes.c_int64 * 3)(*t.stride()[:3])


def make_shape(q: torch.Tensor, k_cache: Optional[torch.Tensor] = None, k_tree: Optional[torch.Tensor] = None,
               H_kv: Optional[int] = None, N_max: Optional[int] = None, scale: Optional[float] = None,
               num_splits: int = 0, max_seqlen: int = 0) -> hta_shape_t:
    """hta_shape_t from q [B,T,H,d], k_cache [B,N,H_kv,d], k_tree [B,T,H_kv,d] (strides included)."""
    B, T, H, d = q.shape
    s = hta_shape_t()
    s.B, s.T, s.H, s.d = B, T, H, d
    if k_cache is not None:
        s.N_max, s.H_kv = k_cache.shape[1], k_cache.shape[2]
        s.kv_strides = _strides3(k_cache)
    else:
        s.N_max = N_max or 0
        s.H_kv = H_kv if H_kv is not None else (k_tree.shape[2] if k_tree is not None else H)
    if k_tree is not None:
        s.tkv_strides = _strides3(k_tree)
        s.H_kv = k_tree.shape[2]
    s.softmax_scale = float(scale) if scale is not None else 1.0 / d ** 0.5
    s.dtype = _dtype_code(q.dtype)
    s.q_strides = _strides3(q)
    s.num_splits = num_splits
    s.max_seqlen = max_seqlen
    return s


def workspace_size(shape: hta_shape_t, num_sms: int = 0) -> int:
    n = lib().hta_workspace_size(ctypes.byref(shape), num_sms)
    if n == ctypes.c_size_t(-1).value:
        raise HtaError("hta_workspace_size", 1)
    return n


def _num_sms(dev) -> int:
    return torch.cuda.get_device_properties(dev).multi_processor_count


def new_workspace(shape: hta_shape_t, device) -> torch.Tensor:
    """A (zero-filled) workspace for hta_forward / hta_prefix_attn of this shape."""
    return torch.zeros(max(workspace_size(shape, _num_sms(device)), 16), dtype=torch.uint8, device=device)


def _workspace(shape: hta_shape_t, device, ws: Optional[torch.Tensor]) -> torch.Tensor:
    """The caller's workspace as given (libhta checks its size), else a new zero-filled one."""
    return new_workspace(shape, device) if ws is None else ws


def _hold(stream, *temps):
    """Temporaries created here whose pointers were enqueued on a caller-given `stream`: mark them
    in use on that stream, so the caching allocator does not hand their memory to other work
    before the kernels have run."""
    if stream is None:
        return
    for t in temps:
        if t is not None and t.is_cuda:
            t.record_stream(stream)


def _out_like_q(q: torch.Tensor, o: Optional[torch.Tensor]) -> torch.Tensor:
    """The ABI writes O with q's strides (hta_shape_t.q_strides): allocate it that way."""
    if o is None:
        return torch.empty_strided(q.shape, q.stride(), dtype=q.dtype, device=q.device)
    if o.shape != q.shape or o.stride() != q.stride() or o.dtype != q.dtype:
        raise ValueError("o must have q's shape, strides and dtype")
    return o


# --------------------------------------------------------------------------- attention

def hta_prefix_attn(q, k_cache, v_cache, cache_seqlens=None, o_part=None, lse_part=None, ws=None,
                    scale=None, num_splits=0, max_seqlen=0, stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Unmasked prefix pass: fp32 O [B,T,H,d] and natural-log LSE [B,H,T]."""
    shape = make_shape(q, k_cache=k_cache, scale=scale, num_splits=num_splits, max_seqlen=max_seqlen)
    B, T, H, d = q.shape
    if o_part is None:
        o_part = torch.empty(B, T, H, d, dtype=torch.float32, device=q.device)
    if lse_part is None:
        lse_part = torch.empty(B, H, T, dtype=torch.float32, device=q.device)
    ws_given = ws
    ws = _workspace(shape, q.device, ws)
    _check("hta_prefix_attn", lib().hta_prefix_attn(ctypes.byref(shape), _ptr(q), _ptr(k_cache), _ptr(v_cache),
                                                    _ptr(cache_seqlens), _ptr(o_part), _ptr(lse_part), _ptr(ws),
                                                    ws.numel() * ws.element_size(), _stream(stream)))
    _hold(stream, None if ws is ws_given else ws)
    return o_part, lse_part


def hta_tree_attn(q, k_tree, v_tree, mask, o_part=None, lse_part=None, scale=None,
                  stream=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Masked tree pass.  mask uint8 [B,T,T] or [T,T] (shared by the batch)."""
    shape = make_shape(q, k_tree=k_tree, scale=scale)
    B, T, H, d = q.shape
    mbs = 0 if mask.dim() == 2 else mask.stride(0)
    if o_part is None:
        o_part = torch.empty(B, T, H, d, dtype=torch.float32, device=q.device)
    if lse_part is None:
        lse_part = torch.empty(B, H, T, dtype=torch.float32, device=q.device)
    _check("hta_tree_attn", lib().hta_tree_attn(ctypes.byref(shape), _ptr(q), _ptr(k_tree), _ptr(v_tree),
                                                _ptr(mask), mbs, _ptr(o_part), _ptr(lse_part), _stream(stream)))
    return o_part, lse_part


def hta_merge_lse(o_parts, lse_parts, dtype=torch.bfloat16, o=None, lse_out=None, want_lse=True, H_kv=None,
                  stream=None) -> Tuple[torch.Tensor, Optional[torch.Tensor]]:
    """Merge n partials o_parts [n,B,T,H,d] / lse_parts [n,B,H,T] -> O in `dtype` (+ LSE)."""
    n, B, T, H, d = o_parts.shape
    if o is None:
        o = torch.empty(B, T, H, d, dtype=dtype, device=o_parts.device)
    shape = make_shape(o, H_kv=H_kv or H)
    if want_lse and lse_out is None:
        lse_out = torch.empty(B, H, T, dtype=torch.float32, device=o_parts.device)
    oc, lc = o_parts.contiguous(), lse_parts.contiguous()
    _check("hta_merge_lse", lib().hta_merge_lse(ctypes.byref(shape), n, _ptr(oc), _ptr(lc), _ptr(o), _ptr(lse_out),
                                                _stream(stream)))
    _hold(stream, None if oc is o_parts else oc, None if lc is lse_parts else lc)
    return o, lse_out


def hta_forward(q, k_cache, v_cache, k_tree, v_tree, mask, cache_seqlens=None, o=None, lse_out=None, ws=None,
                want_lse=True, scale=None, num_splits=0, max_seqlen=0, stream=None,
                events=None, tree_ready=None) -> Tuple[torch.Tensor, Optional[torch.Tensor]]:
    """Full Hybrid Tree Attention of one layer: O [B,T,H,d] in q.dtype (+ LSE [B,H,T]).
    `events` = (begin, end) torch.cuda.Event pair recorded around the prefix kernel
    (hta_forward_timed); `tree_ready` = a torch.cuda.Event the tree/merge kernel waits for
    (hta_forward_ex: k_tree / v_tree / mask may still be in flight during the prefix pass)."""
    shape = make_shape(q, k_cache=k_cache, k_tree=k_tree, scale=scale, num_splits=num_splits, max_seqlen=max_seqlen)
    B, T, H, d = q.shape
    mbs = 0 if mask.dim() == 2 else mask.stride(0)
    o = _out_like_q(q, o)
    if want_lse and lse_out is None:
        lse_out = torch.empty(B, H, T, dtype=torch.float32, device=q.device)
    ws_given = ws
    ws = _workspace(shape, q.device, ws)
    if tree_ready is not None:
        _check("hta_forward_ex", lib().hta_forward_ex(
            ctypes.byref(shape), _ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(cache_seqlens), _ptr(k_tree),
            _ptr(v_tree), _ptr(mask), mbs, _ptr(o), _ptr(lse_out), _ptr(ws), ws.numel() * ws.element_size(),
            _stream(stream), ctypes.c_void_p(tree_ready.cuda_event)))
    elif events is None:
        _check("hta_forward", lib().hta_forward(ctypes.byref(shape), _ptr(q), _ptr(k_cache), _ptr(v_cache),
                                                _ptr(cache_seqlens), _ptr(k_tree), _ptr(v_tree), _ptr(mask), mbs,
                                                _ptr(o), _ptr(lse_out), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))
    else:
        ev0, ev1 = (ctypes.c_void_p(e.cuda_event) for e in events)
        _check("hta_forward_timed", lib().hta_forward_timed(
            ctypes.byref(shape), _ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(cache_seqlens), _ptr(k_tree),
            _ptr(v_tree), _ptr(mask), mbs, _ptr(o), _ptr(lse_out), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream), ev0, ev1))
    _hold(stream, None if ws is ws_given else ws)
    return o, lse_out


def hta_forward_tree(q, k_cache, v_cache, k_tree, v_tree, parents, cache_seqlens=None, o=None, lse_out=None,
                     ws=None, want_lse=True, scale=None, num_splits=0, max_seqlen=0, stream=None,
                     events=None, tree_ready=None) -> Tuple[torch.Tensor, Optional[torch.Tensor]]:
    """hta_forward with the tree as its parent array (int32 [T] shared, or [B, T]); each row's
    visible tree keys are derived in the kernels (no mask input).  `events` = optional (begin,
    end) torch.cuda.Event pair recorded around the prefix kernel; `tree_ready` = a
    torch.cuda.Event the kernel after the prefix pass waits for (k_tree / v_tree / parents may
    still be in flight)."""
    shape = make_shape(q, k_cache=k_cache, k_tree=k_tree, scale=scale, num_splits=num_splits, max_seqlen=max_seqlen)
    B, T, H, d = q.shape
    par = parents if parents.dtype == torch.int32 and parents.is_contiguous() else parents.to(torch.int32).contiguous()
    pbs = 0 if par.dim() == 1 else par.stride(0)
    o = _out_like_q(q, o)
    if want_lse and lse_out is None:
        lse_out = torch.empty(B, H, T, dtype=torch.float32, device=q.device)
    ws_given = ws
    ws = _workspace(shape, q.device, ws)
    ev0, ev1 = (None, None) if events is None else (ctypes.c_void_p(e.cuda_event) for e in events)
    _check("hta_forward_tree", lib().hta_forward_tree(
        ctypes.byref(shape), _ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(cache_seqlens), _ptr(k_tree), _ptr(v_tree),
        _ptr(par), pbs, _ptr(o), _ptr(lse_out), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream), ev0, ev1,
        None if tree_ready is None else ctypes.c_void_p(tree_ready.cuda_event)))
    _hold(stream, None if ws is ws_given else ws, None if par is parents else par)
    return o, lse_out


def hta_forward_paged(q, k_pool, v_pool, block_table, k_tree, v_tree, mask, cache_seqlens=None, o=None,
                      lse_out=None, ws=None, want_lse=True, scale=None, num_splits=0, max_seqlen=0, stream=None):
    """hta_forward over a paged cache: k_pool/v_pool [num_pages, page_size, H_kv, d] bf16,
    block_table int32 [B, max_pages] (device)."""
    num_pages, page_size, Hkv, d = k_pool.shape
    B, T, H, _ = q.shape
    max_pages = block_table.shape[1]
    shape = make_shape(q, k_tree=k_tree, H_kv=Hkv, N_max=max_pages * page_size, scale=scale, num_splits=num_splits,
                       max_seqlen=max_seqlen)
    shape.N_max = max_pages * page_size
    mbs = 0 if mask.dim() == 2 else mask.stride(0)
    o = _out_like_q(q, o)
    if want_lse and lse_out is None:
        lse_out = torch.empty(B, H, T, dtype=torch.float32, device=q.device)
    ws_given = ws
    ws = _workspace(shape, q.device, ws)
    bt = block_table.to(torch.int32).contiguous()
    _check("hta_forward_paged", lib().hta_forward_paged(
        ctypes.byref(shape), _ptr(q), _ptr(k_pool), _ptr(v_pool), num_pages, page_size, _ptr(bt), max_pages,
        _ptr(cache_seqlens), _ptr(k_tree), _ptr(v_tree), _ptr(mask), mbs, _ptr(o), _ptr(lse_out), _ptr(ws),
        ws.numel() * ws.element_size(), _stream(stream)))
    _hold(stream, None if ws is ws_given else ws, None if bt is block_table else bt)
    return o, lse_out


def _fp8_shape(q, k8, k_tree=None, scale=None, num_splits=0, max_seqlen=0):
    """Shape of an FP8-cache call: k8 is a uint8 (E4M3 bytes) [B, N, H_kv, d] tensor."""
    if k8.dtype not in (torch.uint8, getattr(torch, "float8_e4m3fn", torch.uint8)):
        raise TypeError("the FP8 cache must hold E4M3 bytes (uint8 or float8_e4m3fn)")
    shape = make_shape(q, k_tree=k_tree, H_kv=k8.shape[2], N_max=k8.shape[1], scale=scale, num_splits=num_splits,
                       max_seqlen=max_seqlen)
    shape.N_max, shape.H_kv = k8.shape[1], k8.shape[2]
    shape.kv_strides = _strides3(k8)
    return shape


def hta_forward_fp8kv(q, k8, v8, k_scale, v_scale, k_tree, v_tree, mask, cache_seqlens=None, o=None, lse_out=None,
                      ws=None, want_lse=True, scale=None, num_splits=0, max_seqlen=0, stream=None):
    """hta_forward over an E4M3 cache k8 / v8 [B, N, H_kv, d] (uint8 bytes) with per-KV-head
    float32 scales (K = k_scale[g] * K8, V = v_scale[g] * V8); q / tree K,V / O bf16."""
    shape = _fp8_shape(q, k8, k_tree=k_tree, scale=scale, num_splits=num_splits, max_seqlen=max_seqlen)
    B, T, H, d = q.shape
    mbs = 0 if mask.dim() == 2 else mask.stride(0)
    o = _out_like_q(q, o)
    if want_lse and lse_out is None:
        lse_out = torch.empty(B, H, T, dtype=torch.float32, device=q.device)
    ws_given = ws
    ws = _workspace(shape, q.device, ws)
    ks, vs = k_scale.to(torch.float32).contiguous(), v_scale.to(torch.float32).contiguous()
    _check("hta_forward_fp8kv", lib().hta_forward_fp8kv(
        ctypes.byref(shape), _ptr(q), _ptr(k8), _ptr(v8), _ptr(ks), _ptr(vs), _ptr(cache_seqlens), _ptr(k_tree),
        _ptr(v_tree), _ptr(mask), mbs, _ptr(o), _ptr(lse_out), _ptr(ws), ws.numel() * ws.element_size(),
        _stream(stream)))
    _hold(stream, None if ws is ws_given else ws, None if ks is k_scale else ks, None if vs is v_scale else vs)
    return o, lse_out


def hta_prefix_attn_fp8kv(q, k8, v8, k_scale, v_scale, cache_seqlens=None, o_part=None, lse_part=None, ws=None,
                          scale=None, num_splits=0, max_seqlen=0, stream=None):
    """Prefix pass over an E4M3 cache: fp32 O [B,T,H,d] and natural-log LSE [B,H,T]."""
    shape = _fp8_shape(q, k8, scale=scale, num_splits=num_splits, max_seqlen=max_seqlen)
    B, T, H, d = q.shape
    if o_part is None:
        o_part = torch.empty(B, T, H, d, dtype=torch.float32, device=q.device)
    if lse_part is None:
        lse_part = torch.empty(B, H, T, dtype=torch.float32, device=q.device)
    ws_given = ws
    ws = _workspace(shape, q.device, ws)
    ks, vs = k_scale.to(torch.float32).contiguous(), v_scale.to(torch.float32).contiguous()
    _check("hta_prefix_attn_fp8kv", lib().hta_prefix_attn_fp8kv(
        ctypes.byref(shape), _ptr(q), _ptr(k8), _ptr(v8), _ptr(ks), _ptr(vs), _ptr(cache_seqlens), _ptr(o_part),
        _ptr(lse_part), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))
    _hold(stream, None if ws is ws_given else ws, None if ks is k_scale else ks, None if vs is v_scale else vs)
    return o_part, lse_part


# --------------------------------------------------------------------------- tree utilities

def hta_build_tree_mask(parents: torch.Tensor, mask: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """uint8 [T,T] ancestor mask from int32 parents [T] (device if `parents` is on CUDA)."""
    parents_in = parents
    parents = parents.to(torch.int32).contiguous()
    T = parents.numel()
    if mask is None:
        mask = torch.empty(T, T, dtype=torch.uint8, device=parents.device)
    on_dev = 1 if parents.is_cuda else 0
    _check("hta_build_tree_mask", lib().hta_build_tree_mask(_ptr(parents), T, _ptr(mask), on_dev,
                                                            _stream(stream) if on_dev else None))
    _hold(stream, None if parents is parents_in else parents)
    return mask


def hta_validate_tree_mask(mask: torch.Tensor) -> bool:
    m = mask.to("cpu", torch.uint8).contiguous()
    rc = lib().hta_validate_tree_mask(_ptr(m), m.shape[0])
    if rc not in (0, 3):
        _check("hta_validate_tree_mask", rc)
    return rc == 0


def hta_accept_greedy(parents, draft_tokens, target_argmax, root: int = 0, context_argmax: int = -1,
                      path=None, path_len=None, bonus=None, stream=None):
    """Greedy accepted path.  Host tensors -> (list path, int bonus); CUDA tensors -> device
    tensors (path int32 [T], path_len int32 [1], bonus int32 [1]) without synchronising."""
    given = (parents, draft_tokens, target_argmax)
    parents = parents.to(torch.int32).contiguous()
    draft_tokens = draft_tokens.to(torch.int32).contiguous()
    target_argmax = target_argmax.to(torch.int32).contiguous()
    T = parents.numel()
    dev = parents.device
    path = torch.empty(T, dtype=torch.int32, device=dev) if path is None else path
    path_len = torch.empty(1, dtype=torch.int32, device=dev) if path_len is None else path_len
    bonus = torch.empty(1, dtype=torch.int32, device=dev) if bonus is None else bonus
    on_dev = 1 if parents.is_cuda else 0
    _check("hta_accept_greedy", lib().hta_accept_greedy(_ptr(parents), _ptr(draft_tokens), _ptr(target_argmax), T,
                                                        root, context_argmax, _ptr(path), _ptr(path_len), _ptr(bonus),
                                                        on_dev, _stream(stream) if on_dev else None))
    if on_dev:
        _hold(stream, *(t for t, g in zip((parents, draft_tokens, target_argmax), given) if t is not g))
        return path, path_len, bonus
    n = int(path_len[0])
    return [int(x) for x in path[:n].tolist()], int(bonus[0])


def hta_tree_step(parents, draft_tokens, target_argmax, root: int = 0, context_argmax: int = -1, mask=None,
                  want_mask=True, path=None, path_len=None, bonus=None, stream=None):
    """a0 + a6 in one device launch: (mask uint8 [T,T] or None, path int32 [T], path_len int32 [1],
    bonus int32 [1]) from CUDA int32 tensors parents / draft_tokens / target_argmax [T]."""
    given = (parents, draft_tokens, target_argmax)
    parents = parents.to(torch.int32).contiguous()
    draft_tokens = draft_tokens.to(torch.int32).contiguous()
    target_argmax = target_argmax.to(torch.int32).contiguous()
    T = parents.numel()
    dev = parents.device
    if want_mask and mask is None:
        mask = torch.empty(T, T, dtype=torch.uint8, device=dev)
    path = torch.empty(T, dtype=torch.int32, device=dev) if path is None else path
    path_len = torch.empty(1, dtype=torch.int32, device=dev) if path_len is None else path_len
    bonus = torch.empty(1, dtype=torch.int32, device=dev) if bonus is None else bonus
    _check("hta_tree_step", lib().hta_tree_step(_ptr(parents), T, _ptr(mask if want_mask else None), _ptr(draft_tokens),
                                                _ptr(target_argmax), root, context_argmax, _ptr(path), _ptr(path_len),
                                                _ptr(bonus), _stream(stream)))
    _hold(stream, *(t for t, g in zip((parents, draft_tokens, target_argmax), given) if t is not g))
    return (mask if want_mask else None), path, path_len, bonus


def hta_commit_kv(path, path_len, k_tree, v_tree, k_cache, v_cache, cache_seqlens, seqlens_out=None,
                  stream=None):
    """Append the accepted tree K/V rows to the cache in path order (device, in place).
    path int32 [B, >= T] (or [T] for B = 1), path_len int32 [B] (or [1]); returns seqlens_out
    (int32 [B], a new tensor unless given; may be cache_seqlens itself)."""
    B, T, Hkv, d = k_tree.shape
    s = hta_shape_t()
    s.B, s.T, s.H, s.H_kv, s.d = B, T, Hkv, Hkv, d
    s.N_max = k_cache.shape[1]
    s.softmax_scale = 1.0
    s.dtype = _dtype_code(k_tree.dtype)
    s.q_strides = (ctypes.c_int64 * 3)(T * Hkv * d, Hkv * d, d)
    s.kv_strides = _strides3(k_cache)
    s.tkv_strides = _strides3(k_tree)
    path = path.to(torch.int32).reshape(B, -1)
    if path.stride(-1) != 1:
        path = path.contiguous()
    path_len = path_len.to(torch.int32).reshape(B)
    if seqlens_out is None:
        seqlens_out = torch.empty(B, dtype=torch.int32, device=k_cache.device)
    _check("hta_commit_kv", lib().hta_commit_kv(ctypes.byref(s), _ptr(path), path.stride(0), _ptr(path_len),
                                                _ptr(k_tree), _ptr(v_tree), _ptr(k_cache), _ptr(v_cache),
                                                _ptr(cache_seqlens), _ptr(seqlens_out), _stream(stream)))
    _hold(stream, path, path_len)
    return seqlens_out


# --------------------------------------------------------------------------- sequence parallel

class HtaComm:
    """NCCL communicator for hta_forward_seqpar (one process per GPU).  Rank 0 creates the
    unique id; it is broadcast with the given torch.distributed process group."""

    def __init__(self, rank: int, world_size: int, group=None):
        import torch.distributed as dist
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            _check("hta_comm_unique_id", lib().hta_comm_unique_id(buf))
            uid = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if world_size > 1:
            t = uid.cuda() if dist.get_backend(group) == "nccl" else uid
            dist.broadcast(t, src=0, group=group)
            uid = t.cpu()
        raw = (ctypes.c_uint8 * 128)(*uid.tolist())
        h = ctypes.c_void_p()
        _check("hta_comm_create", lib().hta_comm_create(raw, world_size, rank, ctypes.byref(h)))
        self.handle, self.rank, self.world_size = h, rank, world_size

    def close(self):
        if self.handle:
            lib().hta_comm_destroy(self.handle)
            self.handle = None

    def workspace_size(self, shape: hta_shape_t) -> int:
        n = lib().hta_workspace_size_seqpar(ctypes.byref(shape), _num_sms(torch.cuda.current_device()),
                                            self.world_size)
        if n == ctypes.c_size_t(-1).value:
            raise HtaError("hta_workspace_size_seqpar", 1)
        return n

    def forward(self, q, k_cache_local, v_cache_local, k_tree, v_tree, mask=None, cache_seqlens_local=None,
                gather_output=False, o=None, lse_out=None, ws=None, want_lse=True, scale=None, num_splits=0,
                stream=None, parents=None):
        """hta_forward_seqpar over this rank's KV slice; the tree as `mask`, or as `parents`
        (int32 [T] shared or [B, T]: hta_forward_seqpar_tree)."""
        if (mask is None) == (parents is None):
            raise ValueError("give exactly one of mask and parents")
        shape = make_shape(q, k_cache=k_cache_local, k_tree=k_tree, scale=scale, num_splits=num_splits)
        B, T, H, d = q.shape
        Hx = H if gather_output else H // self.world_size
        if o is None:
            o = torch.empty(B, T, Hx, d, dtype=q.dtype, device=q.device)
        if want_lse and lse_out is None:
            lse_out = torch.empty(B, Hx, T, dtype=torch.float32, device=q.device)
        n = self.workspace_size(shape)
        ws_given = ws
        if ws is None or ws.numel() < n:
            ws = torch.empty(n, dtype=torch.uint8, device=q.device)
        if parents is not None:
            par = parents if parents.dtype == torch.int32 and parents.is_contiguous() else \
                parents.to(torch.int32).contiguous()
            _check("hta_forward_seqpar_tree", lib().hta_forward_seqpar_tree(
                self.handle, ctypes.byref(shape), _ptr(q), _ptr(k_cache_local), _ptr(v_cache_local),
                _ptr(cache_seqlens_local), _ptr(k_tree), _ptr(v_tree), _ptr(par), 0 if par.dim() == 1 else par.stride(0),
                _ptr(o), _ptr(lse_out), 1 if gather_output else 0, _ptr(ws), ws.numel() * ws.element_size(),
                _stream(stream)))
            _hold(stream, None if ws is ws_given else ws, None if par is parents else par)
            return o, lse_out
        mbs = 0 if mask.dim() == 2 else mask.stride(0)
        _check("hta_forward_seqpar", lib().hta_forward_seqpar(
            self.handle, ctypes.byref(shape), _ptr(q), _ptr(k_cache_local), _ptr(v_cache_local),
            _ptr(cache_seqlens_local), _ptr(k_tree), _ptr(v_tree), _ptr(mask), mbs, _ptr(o), _ptr(lse_out),
            1 if gather_output else 0, _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))
        _hold(stream, None if ws is ws_given else ws)
        return o, lse_out

    def enable_p2p(self, shapes, group=None) -> bool:
        """Enable the peer-memory exchange (hta_comm_p2p_*) for steps of the given hta_shape_t's
        (local shapes): allocate this rank's buffers, all-gather the IPC handles over the process
        group, open the peers'.  Returns False (the NCCL exchange stays) if any rank failed."""
        import torch.distributed as dist
        cap = max(seqpar_block_floats(s, self.world_size) for s in shapes)
        buf = (ctypes.c_uint8 * 128)()
        rc = lib().hta_comm_p2p_alloc(self.handle, cap, buf)
        mine = torch.tensor(list(bytes(buf)) + [1 if rc == 0 else 0], dtype=torch.uint8)
        if self.world_size > 1:
            t = mine.cuda() if dist.get_backend(group) == "nccl" else mine
            out = [torch.empty_like(t) for _ in range(self.world_size)]
            dist.all_gather(out, t, group=group)
            every = torch.stack([o.cpu() for o in out])
        else:
            every = mine[None]
        if not bool(every[:, 128].all()):
            return False
        raw = (ctypes.c_uint8 * (128 * self.world_size))(*every[:, :128].flatten().tolist())
        rc = lib().hta_comm_p2p_open(self.handle, raw)
        ok = torch.tensor([1 if rc == 0 else 0], dtype=torch.uint8)
        if self.world_size > 1:  # every rank must have opened its peers
            t = ok.cuda() if dist.get_backend(group) == "nccl" else ok
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
            ok = t.cpu()
        return bool(ok.item())

    def set_p2p(self, enabled: bool) -> None:
        _check("hta_comm_p2p_set", lib().hta_comm_p2p_set(self.handle, 1 if enabled else 0))

    def p2p_error(self) -> bool:
        """True once a final merge gave up waiting for a peer's flag (hta_comm_p2p_error)."""
        return lib().hta_comm_p2p_error(self.handle) != 0

    def async_error(self) -> bool:
        """True if NCCL reported an asynchronous error on this communicator."""
        return lib().hta_comm_async_error(self.handle) != 0


class LoopbackComm:
    """`world_size` virtual ranks of the sequence-parallel step in this process, on the current
    device (hta_comm_create_loopback): every rank's phases run through libhta on one GPU, the
    exchange being device copies.  Used to check the P > 1 data path against the oracle."""

    def __init__(self, world_size: int):
        h = ctypes.c_void_p()
        _check("hta_comm_create_loopback", lib().hta_comm_create_loopback(world_size, ctypes.byref(h)))
        self.handle, self.world_size = h, world_size

    def close(self):
        if self.handle:
            lib().hta_comm_destroy(self.handle)
            self.handle = None

    def workspace_size(self, shape: hta_shape_t) -> int:
        n = lib().hta_workspace_size_seqpar(ctypes.byref(shape), _num_sms(torch.cuda.current_device()),
                                            self.world_size)
        if n == ctypes.c_size_t(-1).value:
            raise HtaError("hta_workspace_size_seqpar", 1)
        return self.world_size * ((n + 15) // 16 * 16)

    def enable_p2p(self, shapes) -> None:
        """The peer-memory exchange between the virtual ranks (hta_comm_p2p_alloc on a loopback
        communicator): every rank's combine writes into the others' receive buffers."""
        cap = max(seqpar_block_floats(s, self.world_size) for s in shapes)
        buf = (ctypes.c_uint8 * 128)()
        _check("hta_comm_p2p_alloc", lib().hta_comm_p2p_alloc(self.handle, cap, buf))

    def forward(self, q, k_slices, v_slices, k_tree, v_tree, mask, seqlens_slices=None, gather_output=False,
                want_lse=True, scale=None, num_splits=0, stream=None):
        """k_slices / v_slices: per-rank KV slices [B, N_r, H_kv, d] (same N_r capacity);
        returns per-rank lists (o, lse) as hta_forward_seqpar would on each rank."""
        P = self.world_size
        assert len(k_slices) == P and len(v_slices) == P
        shape = make_shape(q, k_cache=k_slices[0], k_tree=k_tree, scale=scale, num_splits=num_splits)
        B, T, H, d = q.shape
        Hx = H if gather_output else H // P
        os_ = [torch.empty(B, T, Hx, d, dtype=q.dtype, device=q.device) for _ in range(P)]
        ls = [torch.empty(B, Hx, T, dtype=torch.float32, device=q.device) for _ in range(P)] if want_lse else None
        ws = torch.empty(self.workspace_size(shape), dtype=torch.uint8, device=q.device)
        arr = lambda ts: (ctypes.c_void_p * P)(*[t.data_ptr() for t in ts])
        mbs = 0 if mask.dim() == 2 else mask.stride(0)
        _check("hta_forward_seqpar_loopback", lib().hta_forward_seqpar_loopback(
            self.handle, ctypes.byref(shape), _ptr(q), arr(k_slices), arr(v_slices),
            arr(seqlens_slices) if seqlens_slices is not None else None, _ptr(k_tree), _ptr(v_tree), _ptr(mask),
            mbs, arr(os_), arr(ls) if ls is not None else None, 1 if gather_output else 0, _ptr(ws),
            ws.numel(), _stream(stream)))
        _hold(stream, ws)
        return os_, ls


def seqpar_block_floats(shape: hta_shape_t, world_size: int) -> int:
    """Floats of one rank's exchange block: O [B,T,H/P,d] + LSE [B,H/P,T], rounded to 4."""
    hp = shape.H // world_size
    n = shape.B * shape.T * hp * shape.d + shape.B * hp * shape.T
    return (n + 3) // 4 * 4


def shard_bounds(N: int, world_size: int, rank: int) -> Tuple[int, int]:
    """Contiguous sequence shard [lo, hi) of rank `rank`."""
    return N * rank // world_size, N * (rank + 1) // world_size
