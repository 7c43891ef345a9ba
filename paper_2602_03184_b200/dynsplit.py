"""Thin Python binding of libdynsplit.so (include/dynsplit.h).

Argument marshalling only: tensors are checked for dtype/shape/contiguity,
outputs and workspaces are allocated with torch (device memory plumbing), and
the raw device pointers plus the current CUDA stream go through ctypes to the
C ABI.  Every step of the path runs in the library's CUDA kernels; there is no
fallback -- if the library is missing or no GPU is present the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libdynsplit_debug.so" if os.environ.get("DYNSPLIT_DEBUG_BUILD")
                        else "libdynsplit.so")
if os.environ.get("DYNSPLIT_LIB_AB"):  # A/B timing of another in-tree build (tools/); never set by the tests
    LIB_PATH = os.path.join(_PKG, "lib", os.environ["DYNSPLIT_LIB_AB"])

OK = 0
BF16, FP32 = 0, 1
(OP_SCORE_DELIMITERS, OP_SEGMENT, OP_BUILD_BLOCKS, OP_SELECT, OP_DECODE_ATTN, OP_DECODE_LAYER,
 OP_APPEND, OP_MAP_PAGES, OP_REPACK, OP_REUSE, OP_DECODE_OFFLOAD) = range(11)
# device error word bits (include/dynsplit.h DYNSPLIT_DEVERR_*)
DEVERR_PLAN_COVERAGE, DEVERR_PLAN_MISMATCH, DEVERR_PAGE_CAPACITY = 1, 2, 4
DEVERR_SELECT_OVERFLOW, DEVERR_BLOCK_TOO_LONG, DEVERR_SYNC_TIMEOUT = 8, 16, 32
INT32_MAX = 0x7FFFFFFF


class DynsplitError(RuntimeError):
    pass


class Shape(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("S", ctypes.c_int32), ("Hq", ctypes.c_int32),
                ("Hkv", ctypes.c_int32), ("d", ctypes.c_int32),
                ("n_score_layers", ctypes.c_int32), ("kv_dtype", ctypes.c_int32)]


class Config(ctypes.Structure):
    _fields_ = [("W", ctypes.c_int32), ("R", ctypes.c_int32), ("alpha_pen", ctypes.c_float),
                ("C", ctypes.c_int32), ("delta", ctypes.c_int32), ("lambda_num", ctypes.c_int32),
                ("lambda_den", ctypes.c_int32), ("page_size", ctypes.c_int32),
                ("digest_mode", ctypes.c_int32), ("page_cap", ctypes.c_int32),
                ("gqa_mode", ctypes.c_int32), ("budget_mode", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class KVCache(ctypes.Structure):
    """dynsplit_kv_cache (include/dynsplit.h, NEXT-3)."""
    _fields_ = [("n_slots", ctypes.c_int32), ("slot_page", ctypes.c_void_p), ("Kc", ctypes.c_void_p),
                ("Vc", ctypes.c_void_p), ("fetch", ctypes.c_void_p), ("fetch_count", ctypes.c_void_p),
                ("reuse_stats", ctypes.c_void_p), ("reuse_len", ctypes.c_void_p),
                ("worklist_cache", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I = ctypes.c_int32
_SZ = ctypes.c_size_t
_PS = ctypes.POINTER(Shape)
_PC = ctypes.POINTER(Config)

# name -> (restype, argtypes); every symbol declared in include/dynsplit.h
SIGNATURES = {
    "dynsplit_default_config": (None, [_PC]),
    "dynsplit_max_blocks": (_I, [_I, _PC]),
    "dynsplit_max_pages": (_I, [_I, _PC]),
    "dynsplit_max_selected": (_I, [_I, _I, _PC]),
    "dynsplit_worklist_bytes": (_SZ, [_PS, _PC, _I]),
    "dynsplit_workspace_bytes": (_SZ, [_I, _PS, _PC, _I]),
    "dynsplit_status_string": (ctypes.c_char_p, [_I]),
    "dynsplit_version": (ctypes.c_char_p, []),
    "dynsplit_last_error": (ctypes.c_char_p, []),
    "dynsplit_read_device_error": (_I, [_P, _P]),
    "dynsplit_clear_device_error": (_I, [_P, _P]),
    "dynsplit_stream_fence": (_I, [_P]),
    "dynsplit_score_delimiters": (_I, [_PS, _PC, _P, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_weight_table": (_I, [_PS, _P, _P, _I, _P, _P, _P]),
    "dynsplit_segment": (_I, [_PS, _PC, _P, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_map_pages": (_I, [_PS, _PC, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_repack_digest": (_I, [_PS, _PC, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_build_blocks": (_I, [_PS, _PC, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                   _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_score_blocks": (_I, [_PS, _PC, _P, _P, _P, _P, _P]),
    "dynsplit_select_from_scores": (_I, [_PS, _PC, _I, _P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P,
                                         _P, _SZ, _P]),
    "dynsplit_select": (_I, [_PS, _PC, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_decode_attn": (_I, [_PS, _PC, _P, _P, _P, _P, _P, _P, ctypes.c_float, _P, _P, _P,
                                  _SZ, _P]),
    "dynsplit_decode_layer": (_I, [_PS, _PC, _I, _P, _P, _P, _P, _P, _P, _P, ctypes.c_float, _P, _P,
                                   _P, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_append_plan": (_I, [_PS, _PC, _I, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_append_kv": (_I, [_PS, _PC, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dynsplit_append_kv_layers": (_I, [_PS, _PC, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dynsplit_merge_partials": (_I, [_P, _P, _I, _I, _I, _P, _P, _P]),
    "dynsplit_append_plan_dev": (_I, [_PS, _PC, _P, _I, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_append_kv_layers_dev": (_I, [_PS, _PC, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "dynsplit_step_host_workspace_bytes": (_SZ, [_PS, _PC, _I]),
    "dynsplit_decode_step_host": (_I, [_PS, _PC, _I, _P, _P, _P, _P, _P, _P, _P, _P,
                                       ctypes.c_float, _P, _P, _P, _P, _SZ, _P]),
    "dynsplit_cache_slots": (_I, [_PS, _PC, _I]),
    "dynsplit_reuse_plan": (_I, [_PS, _PC, _P, _I, _I, ctypes.POINTER(KVCache), _P, _SZ, _P]),
    "dynsplit_fetch_pages": (_I, [_PS, _PC, _P, _P, _P, _P, _I, ctypes.POINTER(KVCache), _P]),
    "dynsplit_decode_layer_offload": (_I, [_PS, _PC, _I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I,
                                           ctypes.POINTER(KVCache), ctypes.c_float, _P, _P, _P, _P, _P, _P,
                                           _P, _SZ, _P]),
    "dynsplit_step_host_layers_workspace_bytes": (_SZ, [_PS, _PC, _I, _I]),
    "dynsplit_decode_step_host_layers": (_I, [_PS, _PC, _I, _I, _P, _P, _P, _P, _P, _P, _P,
                                              ctypes.c_float, _P, _P, _P, _P, _SZ, _P]),
}

_lib = None


def lib():
    """Load libdynsplit.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DynsplitError(f"{LIB_PATH} missing: run `python -m paper_2602_03184_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def read_device_error(ws: torch.Tensor) -> int:
    """Synchronise the current stream and return the device error word of a
    workspace (DEVERR_* bits; 0 = no data-dependent error)."""
    v = lib().dynsplit_read_device_error(_ptr(ws), _stream(ws.device))
    if v < 0:
        raise DynsplitError("dynsplit_read_device_error failed")
    return int(v)


def clear_device_error(ws: torch.Tensor) -> None:
    _check(lib().dynsplit_clear_device_error(_ptr(ws), _stream(ws.device)), "clear_device_error")


def stream_fence(device=None) -> None:
    """dynsplit_stream_fence on the current stream (see include/dynsplit.h)."""
    _check(lib().dynsplit_stream_fence(_stream(device)), "stream_fence")


def _check(st: int, what: str):
    if st != OK:
        msg = lib().dynsplit_status_string(st).decode()
        detail = lib().dynsplit_last_error().decode() if st == 6 else ""
        raise DynsplitError(f"{what}: {msg} ({st}) {detail}".rstrip())


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise DynsplitError("expected a CUDA tensor (the library has no CPU path)")
    if not t.is_contiguous():
        raise DynsplitError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return FP32
    raise DynsplitError(f"unsupported KV dtype {t.dtype}")


def default_config(**overrides) -> Config:
    c = Config()
    lib().dynsplit_default_config(ctypes.byref(c))
    for k, v in overrides.items():
        setattr(c, k, v)
    return c


def make_shape(B, S, Hq, Hkv, d=128, n_score_layers=1, kv_dtype=BF16) -> Shape:
    return Shape(B, S, Hq, Hkv, d, n_score_layers, kv_dtype)


def max_blocks(S: int, cfg: Config) -> int:
    return lib().dynsplit_max_blocks(S, ctypes.byref(cfg))


def max_pages(S: int, cfg: Config) -> int:
    return lib().dynsplit_max_pages(S, ctypes.byref(cfg))


def max_selected(budget: int, S: int, cfg: Config) -> int:
    return lib().dynsplit_max_selected(budget, S, ctypes.byref(cfg))


def workspace_bytes(op: int, shape: Shape, cfg: Config, budget: int = 1) -> int:
    return lib().dynsplit_workspace_bytes(op, ctypes.byref(shape), ctypes.byref(cfg), budget)


def worklist_bytes(shape: Shape, cfg: Config, budget: int) -> int:
    return lib().dynsplit_worklist_bytes(ctypes.byref(shape), ctypes.byref(cfg), budget)


_WS = {}


def workspace(nbytes: int, device, key: str) -> torch.Tensor:
    """Zero-initialised, cached device workspace (the library keeps its
    counters zeroed between calls, so a workspace is reusable on one stream)."""
    dev = torch.device(device)
    k = (dev.index, key)
    t = _WS.get(k)
    if t is None or t.numel() < nbytes:
        t = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _WS[k] = t
    return t


# ---------------------------------------------------------------------------
# prefill
# ---------------------------------------------------------------------------
@dataclass
class PagedLayer:
    """Output of block construction for one layer (plan + pages + digests)."""
    shape: Shape
    cfg: Config
    w10: torch.Tensor          # uint8 [B, n_ids]
    block_starts: torch.Tensor  # int32 [B, max_blocks+1]
    n_blocks: torch.Tensor     # int32 [B]
    page_first: torch.Tensor   # int32 [B, max_blocks+1]
    page_block: torch.Tensor   # int32 [B, max_pages]
    page_valid: torch.Tensor   # int16 [B, max_pages]
    n_pages: torch.Tensor      # int32 [B]
    Kp: Optional[torch.Tensor]  # [B, Hkv, max_pages, P, d]
    Vp: Optional[torch.Tensor]
    digests: Optional[torch.Tensor]  # [B, Hkv, max_blocks, 2, d]
    delim_scores: Optional[torch.Tensor] = None


def score_delimiters(tokens, delim_ids, Qs, Ks, cfg: Config):
    """Row a1 (Alg. 1).  tokens int32 [B,S]; Qs bf16 [Ls,B,S,Hq,d]; Ks [Ls,B,S,Hkv,d]."""
    Ls, B, S, Hq, d = Qs.shape
    shape = make_shape(B, S, Hq, Ks.shape[3], d, Ls, _dtype_code(Qs))
    out = torch.empty(B, S, dtype=torch.float32, device=tokens.device)
    nb = workspace_bytes(OP_SCORE_DELIMITERS, shape, cfg)
    ws = workspace(nb, tokens.device, "score")
    _check(lib().dynsplit_score_delimiters(ctypes.byref(shape), ctypes.byref(cfg), _ptr(tokens),
                                           _ptr(delim_ids), delim_ids.numel(), _ptr(Qs), _ptr(Ks),
                                           _ptr(out), _ptr(ws), ws.numel(), _stream()),
           "score_delimiters")
    return out


def weight_table(tokens, delim_ids, scores):
    """Row a2.  -> uint8 [B, n_ids] weights in tenths."""
    B, S = tokens.shape
    shape = make_shape(B, S, 1, 1)
    w10 = torch.empty(B, delim_ids.numel(), dtype=torch.uint8, device=tokens.device)
    _check(lib().dynsplit_weight_table(ctypes.byref(shape), _ptr(tokens), _ptr(delim_ids),
                                       delim_ids.numel(), _ptr(scores), _ptr(w10), _stream()),
           "weight_table")
    return w10


def segment(tokens, delim_ids, w10, cfg: Config):
    """Row a3 (DD-Select).  -> (block_starts [B, maxb+1], n_blocks [B])."""
    B, S = tokens.shape
    shape = make_shape(B, S, 1, 1)
    mb = max_blocks(S, cfg)
    bs = torch.empty(B, mb + 1, dtype=torch.int32, device=tokens.device)
    nb = torch.empty(B, dtype=torch.int32, device=tokens.device)
    ws = workspace(workspace_bytes(OP_SEGMENT, shape, cfg), tokens.device, "segment")
    _check(lib().dynsplit_segment(ctypes.byref(shape), ctypes.byref(cfg), _ptr(tokens),
                                  _ptr(delim_ids), delim_ids.numel(), _ptr(w10), _ptr(bs), _ptr(nb),
                                  _ptr(ws), ws.numel(), _stream()), "segment")
    return bs, nb


def map_pages(block_starts, n_blocks, S: int, cfg: Config, ws=None):
    """Row a4 part 1.  -> (page_first, page_block, page_valid, n_pages).
    ws: optional OP_MAP_PAGES workspace (device error word)."""
    B = block_starts.shape[0]
    shape = make_shape(B, S, 1, 1)
    mb, mp = max_blocks(S, cfg), max_pages(S, cfg)
    dev = block_starts.device
    pf = torch.empty(B, mb + 1, dtype=torch.int32, device=dev)
    pb = torch.empty(B, mp, dtype=torch.int32, device=dev)
    pv = torch.empty(B, mp, dtype=torch.int16, device=dev)
    npg = torch.empty(B, dtype=torch.int32, device=dev)
    _check(lib().dynsplit_map_pages(ctypes.byref(shape), ctypes.byref(cfg), _ptr(block_starts),
                                    _ptr(n_blocks), _ptr(pf), _ptr(pb), _ptr(pv), _ptr(npg),
                                    _ptr(ws), ws.numel() if ws is not None else 0, _stream()), "map_pages")
    return pf, pb, pv, npg


def repack_digest(K, V, block_starts, n_blocks, page_first, cfg: Config, out=None, ws=None):
    """Row a4 part 2.  K, V [B,S,Hkv,d] -> (Kp, Vp, digests).
    ws: optional OP_REPACK workspace (device error word)."""
    B, S, Hkv, d = K.shape
    shape = make_shape(B, S, Hkv, Hkv, d, 1, _dtype_code(K))
    mb, mp, P = max_blocks(S, cfg), max_pages(S, cfg), cfg.page_size
    if out is None:
        Kp = torch.empty(B, Hkv, mp, P, d, dtype=K.dtype, device=K.device)
        Vp = torch.empty_like(Kp)
        dig = torch.empty(B, Hkv, mb, 2, d, dtype=K.dtype, device=K.device)
    else:
        Kp, Vp, dig = out
    _check(lib().dynsplit_repack_digest(ctypes.byref(shape), ctypes.byref(cfg), _ptr(K), _ptr(V),
                                        _ptr(block_starts), _ptr(n_blocks), _ptr(page_first),
                                        _ptr(Kp), _ptr(Vp), _ptr(dig), _ptr(ws),
                                        ws.numel() if ws is not None else 0, _stream()), "repack_digest")
    return Kp, Vp, dig


def build_blocks(tokens, delim_ids, K, V, cfg: Config, static_w10=None, Qs=None, Ks=None,
                 Hq: Optional[int] = None, return_scores: bool = False,
                 Hkv: Optional[int] = None) -> PagedLayer:
    """Rows a1-a4 through dynsplit_build_blocks (one C call).

    static_w10: host uint8 sequence (e.g. Table 7) -> static mode; else Qs/Ks
    (bf16 [Ls,B,S,H*,d]) drive the dynamic scoring.  K/V may be None (plan only).
    """
    B, S = tokens.shape
    dev = tokens.device
    if K is not None:
        Hkv, d = K.shape[2], K.shape[3]
        dt = _dtype_code(K)
    else:
        d, dt = 128, BF16
        if Hkv is None:
            Hkv = Ks.shape[3] if Ks is not None else (Hq or 1)
    if Hq is None:
        Hq = Qs.shape[3] if Qs is not None else Hkv
    Ls = Qs.shape[0] if Qs is not None else 1
    shape = make_shape(B, S, Hq, Hkv, d, Ls, dt)
    mb, mp, P = max_blocks(S, cfg), max_pages(S, cfg), cfg.page_size
    n_ids = delim_ids.numel()
    w10 = torch.empty(B, n_ids, dtype=torch.uint8, device=dev)
    bs = torch.empty(B, mb + 1, dtype=torch.int32, device=dev)
    nb = torch.empty(B, dtype=torch.int32, device=dev)
    pf = torch.empty(B, mb + 1, dtype=torch.int32, device=dev)
    pb = torch.empty(B, mp, dtype=torch.int32, device=dev)
    pv = torch.empty(B, mp, dtype=torch.int16, device=dev)
    npg = torch.empty(B, dtype=torch.int32, device=dev)
    scores = torch.empty(B, S, dtype=torch.float32, device=dev) if (return_scores and static_w10 is None) else None
    Kp = Vp = dig = None
    if K is not None:
        Kp = torch.empty(B, Hkv, mp, P, d, dtype=K.dtype, device=dev)
        Vp = torch.empty_like(Kp)
        dig = torch.empty(B, Hkv, mb, 2, d, dtype=K.dtype, device=dev)
    hostw = None
    if static_w10 is not None:
        arr = (ctypes.c_uint8 * n_ids)(*[int(x) for x in static_w10])
        hostw = ctypes.cast(arr, ctypes.c_void_p)
    ws = workspace(workspace_bytes(OP_BUILD_BLOCKS, shape, cfg), dev, "build")
    _check(lib().dynsplit_build_blocks(
        ctypes.byref(shape), ctypes.byref(cfg), _ptr(tokens), _ptr(delim_ids), n_ids, hostw,
        _ptr(Qs), _ptr(Ks), _ptr(K), _ptr(V), _ptr(w10), _ptr(scores), _ptr(bs), _ptr(nb),
        _ptr(pf), _ptr(pb), _ptr(pv), _ptr(npg), _ptr(Kp), _ptr(Vp), _ptr(dig), _ptr(ws),
        ws.numel(), _stream()), "build_blocks")
    return PagedLayer(shape, cfg, w10, bs, nb, pf, pb, pv, npg, Kp, Vp, dig, scores)


# ---------------------------------------------------------------------------
# decode
# ---------------------------------------------------------------------------
# ---------------------------------------------------------------------------
# NEXT-1: growing sequences (decode-time append, incremental DD-Select)
# ---------------------------------------------------------------------------
def alloc_paged(B: int, S_cap: int, Hq: int, Hkv: int, cfg: Config, w10, dtype=torch.bfloat16,
                device="cuda", plan_from: Optional[PagedLayer] = None) -> PagedLayer:
    """Empty paged layer with room for S_cap tokens per sequence (its shape.S
    is the capacity).  w10: uint8 [B, n_ids] device weights.  plan_from: share
    the plan tensors of another layer (the plan is per sequence, not per layer)."""
    d = 128
    shape = make_shape(B, S_cap, Hq, Hkv, d, 1, BF16 if dtype == torch.bfloat16 else FP32)
    mb, mp, P = max_blocks(S_cap, cfg), max_pages(S_cap, cfg), cfg.page_size
    dev = torch.device(device)
    if plan_from is None:
        bs = torch.zeros(B, mb + 1, dtype=torch.int32, device=dev)
        nb = torch.zeros(B, dtype=torch.int32, device=dev)
        pf = torch.zeros(B, mb + 1, dtype=torch.int32, device=dev)
        pb = torch.full((B, mp), -1, dtype=torch.int32, device=dev)
        pv = torch.zeros(B, mp, dtype=torch.int16, device=dev)
        npg = torch.zeros(B, dtype=torch.int32, device=dev)
    else:
        p = plan_from
        bs, nb, pf, pb, pv, npg = p.block_starts, p.n_blocks, p.page_first, p.page_block, p.page_valid, p.n_pages
    Kp = torch.zeros(B, Hkv, mp, P, d, dtype=dtype, device=dev)
    Vp = torch.zeros_like(Kp)
    dig = torch.zeros(B, Hkv, mb, 2, d, dtype=dtype, device=dev)
    return PagedLayer(shape, cfg, w10, bs, nb, pf, pb, pv, npg, Kp, Vp, dig)


def append_workspace(layer: PagedLayer) -> torch.Tensor:
    return torch.zeros(max(workspace_bytes(OP_APPEND, layer.shape, layer.cfg), 256), dtype=torch.uint8,
                       device=layer.block_starts.device)


def append_plan(tokens, delim_ids, layer: PagedLayer, L_prev: int, L: int, ws) -> None:
    """dynsplit_append_plan: re-plan the tail for L_prev -> L tokens (in place)."""
    _check(lib().dynsplit_append_plan(
        ctypes.byref(layer.shape), ctypes.byref(layer.cfg), L_prev, L, _ptr(tokens), _ptr(delim_ids),
        delim_ids.numel(), _ptr(layer.w10), _ptr(layer.block_starts), _ptr(layer.n_blocks),
        _ptr(layer.page_first), _ptr(layer.page_block), _ptr(layer.page_valid), _ptr(layer.n_pages),
        _ptr(ws), ws.numel(), _stream()), "append_plan")


def append_kv(layer: PagedLayer, K_new, V_new, L_prev: int, L: int, ws) -> None:
    """dynsplit_append_kv: move the re-planned rows and write K_new / V_new
    [B, L - L_prev, Hkv, d] into the layer's pages and digests."""
    _check(lib().dynsplit_append_kv(
        ctypes.byref(layer.shape), ctypes.byref(layer.cfg), L_prev, L, _ptr(K_new), _ptr(V_new),
        _ptr(layer.block_starts), _ptr(layer.n_blocks), _ptr(layer.page_first), _ptr(ws),
        _ptr(layer.Kp), _ptr(layer.Vp), _ptr(layer.digests), _stream()), "append_kv")


def append_kv_layers(layers, K_new, V_new, L_prev: int, L: int, ws) -> None:
    """dynsplit_append_kv_layers: append to several layers sharing one plan in one launch."""
    n = len(layers)
    arr = lambda xs: (ctypes.c_void_p * n)(*[ctypes.c_void_p(x.data_ptr()) if x is not None else None
                                             for x in xs])
    lay = layers[0]
    _check(lib().dynsplit_append_kv_layers(
        ctypes.byref(lay.shape), ctypes.byref(lay.cfg), L_prev, L, n, arr(K_new), arr(V_new),
        _ptr(lay.block_starts), _ptr(lay.n_blocks), _ptr(lay.page_first), _ptr(ws),
        arr([x.Kp for x in layers]), arr([x.Vp for x in layers]), arr([x.digests for x in layers]),
        _stream()), "append_kv_layers")


def append_plan_dev(tokens, delim_ids, layer: PagedLayer, L_prev_dev, n_new: int, ws) -> None:
    """dynsplit_append_plan_dev: as append_plan with L_prev read from the
    device int32 tensor L_prev_dev (graph-capturable decode loops)."""
    _check(lib().dynsplit_append_plan_dev(
        ctypes.byref(layer.shape), ctypes.byref(layer.cfg), _ptr(L_prev_dev), n_new, _ptr(tokens), _ptr(delim_ids),
        delim_ids.numel(), _ptr(layer.w10), _ptr(layer.block_starts), _ptr(layer.n_blocks),
        _ptr(layer.page_first), _ptr(layer.page_block), _ptr(layer.page_valid), _ptr(layer.n_pages),
        _ptr(ws), ws.numel(), _stream()), "append_plan_dev")


def append_kv_layers_dev(layers, K_new, V_new, L_prev_dev, n_new: int, ws) -> None:
    """dynsplit_append_kv_layers_dev: as append_kv_layers with L_prev on the device."""
    n = len(layers)
    arr = lambda xs: (ctypes.c_void_p * n)(*[ctypes.c_void_p(x.data_ptr()) for x in xs])
    lay = layers[0]
    _check(lib().dynsplit_append_kv_layers_dev(
        ctypes.byref(lay.shape), ctypes.byref(lay.cfg), _ptr(L_prev_dev), n_new, n, arr(K_new), arr(V_new),
        _ptr(lay.block_starts), _ptr(lay.n_blocks), _ptr(lay.page_first), _ptr(ws),
        arr([x.Kp for x in layers]), arr([x.Vp for x in layers]), arr([x.digests for x in layers]),
        _stream()), "append_kv_layers_dev")


@dataclass
class Selection:
    sel_blocks: torch.Tensor    # int32 [B, Hq, max_sel] (ascending; first n_sel valid)
    n_sel: torch.Tensor         # int32 [B, Hq]
    marginal_block: torch.Tensor  # int32 [B, Hq]
    marginal_keep: torch.Tensor   # int32 [B, Hq]
    worklist: torch.Tensor      # opaque uint8
    scores: Optional[torch.Tensor] = None  # fp32 [B, Hq, max_blocks]


def _decode_shape(q, layer: PagedLayer) -> Shape:
    B, Hq, d = q.shape
    s = layer.shape
    code = _dtype_code(q)
    for name in ("Kp", "Vp", "digests"):
        t = getattr(layer, name)
        if t is not None and _dtype_code(t) != code:
            raise DynsplitError(f"q is {q.dtype} but layer.{name} is {t.dtype}: the KV dtype must match")
    return make_shape(B, s.S, Hq, s.Hkv, d, 1, code)


def score_blocks(q, layer: PagedLayer, out=None):
    """Row a5.  q [B,Hq,d] -> fp32 [B,Hq,max_blocks]."""
    shape = _decode_shape(q, layer)
    mb = max_blocks(shape.S, layer.cfg)
    sc = out if out is not None else torch.empty(shape.B, shape.Hq, mb, dtype=torch.float32, device=q.device)
    _check(lib().dynsplit_score_blocks(ctypes.byref(shape), ctypes.byref(layer.cfg), _ptr(q),
                                       _ptr(layer.digests), _ptr(layer.n_blocks), _ptr(sc),
                                       _stream()), "score_blocks")
    return sc


def _sel_outputs(shape: Shape, cfg: Config, budget: int, dev, want_blocks=True):
    ms = max_selected(budget, shape.S, cfg)
    sb = torch.empty(shape.B, shape.Hq, ms, dtype=torch.int32, device=dev) if want_blocks else None
    ns = torch.empty(shape.B, shape.Hq, dtype=torch.int32, device=dev)
    mg = torch.empty_like(ns)
    kp = torch.empty_like(ns)
    wl = torch.empty(worklist_bytes(shape, cfg, budget), dtype=torch.uint8, device=dev)
    return sb, ns, mg, kp, wl


def select_from_scores(scores, layer: PagedLayer, budget: int, Hq: int, blk_lo: int = 0,
                       blk_hi: int = INT32_MAX, out=None, ws=None) -> Selection:
    """Row a6 on given block scores (seq-split shards pass their block range)."""
    s = layer.shape
    shape = make_shape(s.B, s.S, Hq, s.Hkv, s.d, 1, s.kv_dtype)
    sb, ns, mg, kp, wl = out if out is not None else _sel_outputs(shape, layer.cfg, budget, scores.device)
    if ws is None:
        ws = workspace(workspace_bytes(OP_SELECT, shape, layer.cfg, budget), scores.device, "select")
    _check(lib().dynsplit_select_from_scores(
        ctypes.byref(shape), ctypes.byref(layer.cfg), budget, _ptr(scores), _ptr(layer.block_starts),
        _ptr(layer.n_blocks), _ptr(layer.page_first), blk_lo, blk_hi, _ptr(sb), _ptr(ns), _ptr(mg),
        _ptr(kp), _ptr(wl), _ptr(ws), ws.numel(), _stream()), "select_from_scores")
    return Selection(sb, ns, mg, kp, wl, scores)


def select(q, layer: PagedLayer, budget: int, keep_scores: bool = True, out=None, ws=None) -> Selection:
    """Rows a5 + a6 through dynsplit_select."""
    shape = _decode_shape(q, layer)
    mb = max_blocks(shape.S, layer.cfg)
    if out is None:
        sb, ns, mg, kp, wl = _sel_outputs(shape, layer.cfg, budget, q.device)
        sc = torch.empty(shape.B, shape.Hq, mb, dtype=torch.float32, device=q.device) if keep_scores else None
    else:
        sb, ns, mg, kp, wl, sc = out
    if ws is None:
        ws = workspace(workspace_bytes(OP_SELECT, shape, layer.cfg, budget), q.device, "select")
    _check(lib().dynsplit_select(
        ctypes.byref(shape), ctypes.byref(layer.cfg), budget, _ptr(q), _ptr(layer.digests),
        _ptr(layer.block_starts), _ptr(layer.n_blocks), _ptr(layer.page_first), _ptr(sc), _ptr(sb),
        _ptr(ns), _ptr(mg), _ptr(kp), _ptr(wl), _ptr(ws), ws.numel(), _stream()), "select")
    return Selection(sb, ns, mg, kp, wl, sc)


def decode_attn(q, layer: PagedLayer, worklist: Optional[torch.Tensor], scale: float = 0.0,
                out=None, ws=None):
    """Rows a7 + a8 (worklist=None: dense baseline, row a9).  -> (o fp32 [B,Hq,d], lse fp32 [B,Hq])."""
    shape = _decode_shape(q, layer)
    if out is None:
        o = torch.empty(shape.B, shape.Hq, shape.d, dtype=torch.float32, device=q.device)
        lse = torch.empty(shape.B, shape.Hq, dtype=torch.float32, device=q.device)
    else:
        o, lse = out
    if ws is None:
        ws = workspace(workspace_bytes(OP_DECODE_ATTN, shape, layer.cfg), q.device, "decode")
    _check(lib().dynsplit_decode_attn(
        ctypes.byref(shape), ctypes.byref(layer.cfg), _ptr(q), _ptr(layer.Kp), _ptr(layer.Vp),
        _ptr(layer.page_valid), _ptr(layer.n_pages), _ptr(worklist), ctypes.c_float(scale),
        _ptr(o), _ptr(lse), _ptr(ws), ws.numel(), _stream()), "decode_attn")
    return o, lse


def decode_layer(q, layer: PagedLayer, budget: int, scale: float = 0.0, out=None, ws=None):
    """Rows a5-a8 of one layer through dynsplit_decode_layer (score, select,
    attention in one call).  out = (n_sel, marginal_block,
    marginal_keep, worklist, o, lse) preallocated, or None.
    -> (o, lse, Selection without scores / sel_blocks)."""
    shape = _decode_shape(q, layer)
    if out is None:
        _, ns, mg, kp, wl = _sel_outputs(shape, layer.cfg, budget, q.device, want_blocks=False)
        o = torch.empty(shape.B, shape.Hq, shape.d, dtype=torch.float32, device=q.device)
        lse = torch.empty(shape.B, shape.Hq, dtype=torch.float32, device=q.device)
    else:
        ns, mg, kp, wl, o, lse = out
    if ws is None:
        ws = workspace(workspace_bytes(OP_DECODE_LAYER, shape, layer.cfg, budget), q.device, "layer")
    _check(lib().dynsplit_decode_layer(
        ctypes.byref(shape), ctypes.byref(layer.cfg), budget, _ptr(q), _ptr(layer.digests),
        _ptr(layer.block_starts), _ptr(layer.n_blocks), _ptr(layer.page_first), _ptr(layer.Kp),
        _ptr(layer.Vp), ctypes.c_float(scale), _ptr(ns), _ptr(mg), _ptr(kp), _ptr(wl), _ptr(o),
        _ptr(lse), _ptr(ws), ws.numel(), _stream()), "decode_layer")
    return o, lse, Selection(None, ns, mg, kp, wl, None)


def merge_partials(o_parts, lse_parts, out=None):
    """Row a8 standalone.  o_parts [n, rows, d], lse_parts [n, rows] -> (o [rows, d], lse [rows])."""
    n, rows, d = o_parts.shape
    if out is None:
        o = torch.empty(rows, d, dtype=torch.float32, device=o_parts.device)
        lse = torch.empty(rows, dtype=torch.float32, device=o_parts.device)
    else:
        o, lse = out
    _check(lib().dynsplit_merge_partials(_ptr(o_parts), _ptr(lse_parts), n, rows, d, _ptr(o),
                                         _ptr(lse), _stream()), "merge_partials")
    return o, lse


def decode_step_host(q_host, layer: PagedLayer, budget: int, o_host, lse_host, worklist, ws,
                     scale: float = 0.0):
    """Rows a5-a8 with pinned HOST q/o/lse through dynsplit_decode_step_host."""
    B, Hq, d = q_host.shape
    s = layer.shape
    shape = make_shape(B, s.S, Hq, s.Hkv, d, 1, _dtype_code(q_host))
    for t in (q_host, o_host, lse_host):
        if t.is_cuda or not t.is_pinned():
            raise DynsplitError("decode_step_host expects pinned host tensors")
    _check(lib().dynsplit_decode_step_host(
        ctypes.byref(shape), ctypes.byref(layer.cfg), budget, ctypes.c_void_p(q_host.data_ptr()),
        _ptr(layer.digests), _ptr(layer.block_starts), _ptr(layer.n_blocks), _ptr(layer.page_first),
        _ptr(layer.Kp), _ptr(layer.Vp), _ptr(layer.page_valid), ctypes.c_float(scale),
        ctypes.c_void_p(o_host.data_ptr()), ctypes.c_void_p(lse_host.data_ptr()), _ptr(worklist),
        _ptr(ws), ws.numel(), _stream()), "decode_step_host")


def decode_step_host_layers(q_host, layers, budget: int, o_host, lse_host, worklist, ws, scale: float = 0.0):
    """One token through len(layers) layers with pinned HOST q [L, B, Hq, d]
    and o [L, B, Hq, d] / lse [L, B, Hq] through dynsplit_decode_step_host_layers
    (the layers share one plan)."""
    L, B, Hq, d = q_host.shape
    s = layers[0].shape
    shape = make_shape(B, s.S, Hq, s.Hkv, d, 1, _dtype_code(q_host))
    for t in (q_host, o_host, lse_host):
        if t.is_cuda or not t.is_pinned():
            raise DynsplitError("decode_step_host_layers expects pinned host tensors")
    arr = ctypes.c_void_p * L
    dig = arr(*[lay.digests.data_ptr() for lay in layers])
    kp = arr(*[lay.Kp.data_ptr() for lay in layers])
    vp = arr(*[lay.Vp.data_ptr() for lay in layers])
    lay0 = layers[0]
    _check(lib().dynsplit_decode_step_host_layers(
        ctypes.byref(shape), ctypes.byref(lay0.cfg), budget, L, ctypes.c_void_p(q_host.data_ptr()),
        ctypes.cast(dig, ctypes.c_void_p), _ptr(lay0.block_starts), _ptr(lay0.n_blocks), _ptr(lay0.page_first),
        ctypes.cast(kp, ctypes.c_void_p), ctypes.cast(vp, ctypes.c_void_p), ctypes.c_float(scale),
        ctypes.c_void_p(o_host.data_ptr()), ctypes.c_void_p(lse_host.data_ptr()), _ptr(worklist), _ptr(ws),
        ws.numel(), _stream()), "decode_step_host_layers")


def step_host_layers_workspace_bytes(shape: Shape, cfg: Config, budget: int, n_layers: int) -> int:
    return lib().dynsplit_step_host_layers_workspace_bytes(ctypes.byref(shape), ctypes.byref(cfg), budget, n_layers)


def step_host_workspace_bytes(shape: Shape, cfg: Config, budget: int) -> int:
    return lib().dynsplit_step_host_workspace_bytes(ctypes.byref(shape), ctypes.byref(cfg), budget)


def worklist_rows(worklist: torch.Tensor, shape: Shape, G: int):
    """Host-side reading of a worklist (metrics only): per (b, KV head) the
    number of page entries and of rows streamed (max over the G heads of each
    entry's row count).  Layout: 256-byte header, int32 counts [B*Hkv] padded to
    256 bytes, then 16-byte entries {int32 page, int32 block, uint8 rows[8]},
    interleaved: entry e of (b, KV head) bh at index e * B * Hkv + bh."""
    import numpy as np
    raw = worklist.cpu().numpy()
    nbh = shape.B * shape.Hkv
    hdr = raw[:256].view(np.int32)
    max_wl = int(hdr[1])
    counts = raw[256:256 + 4 * nbh].view(np.int32).copy()
    off = 256 + ((4 * nbh + 255) // 256) * 256
    ent = raw[off: off + 16 * nbh * max_wl].reshape(max_wl, nbh, 16).transpose(1, 0, 2)
    rows = ent[:, :, 8:8 + G].max(axis=2).astype(np.int64)
    streamed = np.array([rows[i, : counts[i]].sum() for i in range(nbh)])
    return counts, streamed


# ---------------------------------------------------------------------------
# NEXT-3: host-offloaded KV with cross-step reuse (Appendix B.2, P:756-765;
# the CPU-GPU deployment)
# ---------------------------------------------------------------------------
def cache_slots(shape: Shape, cfg: Config, budget: int) -> int:
    return lib().dynsplit_cache_slots(ctypes.byref(shape), ctypes.byref(cfg), budget)


@dataclass
class OffloadedLayer:
    """One layer whose pages live in pinned host memory (Kh, Vh [B, Hkv,
    max_pages, P, d]) while the plan, page tables and digests stay resident
    (layer, with Kp = Vp = None), plus the device page cache of n_slots slots
    per (b, KV head) and its per-step outputs (dynsplit_kv_cache)."""
    layer: PagedLayer
    Kh: torch.Tensor
    Vh: torch.Tensor
    n_slots: int
    slot_page: torch.Tensor      # int32 [B, Hkv, n_slots], -1 = empty
    Kc: torch.Tensor             # [B, Hkv, n_slots, P, d]
    Vc: torch.Tensor
    fetch: torch.Tensor          # int32 [B, Hkv, n_slots, 2] (page, slot)
    fetch_count: torch.Tensor    # int32 [B, Hkv]
    reuse_stats: torch.Tensor    # int32 [B, Hkv, 2] (reused, fresh)
    reuse_len: torch.Tensor      # int32 [B]
    worklist_cache: torch.Tensor  # opaque, page = cache slot

    def c(self) -> KVCache:
        p = lambda t: ctypes.c_void_p(t.data_ptr())
        return KVCache(self.n_slots, p(self.slot_page), p(self.Kc), p(self.Vc), p(self.fetch),
                       p(self.fetch_count), p(self.reuse_stats), p(self.reuse_len), p(self.worklist_cache))

    def reset(self) -> None:
        """Empty the cache (the next step moves every page)."""
        self.slot_page.fill_(-1)


def offload_layer(layer: PagedLayer, budget: int, Hq: Optional[int] = None, n_slots: Optional[int] = None,
                  keep_device: bool = False) -> OffloadedLayer:
    """Move a built layer's pages to pinned host memory and allocate its page
    cache (n_slots defaults to dynsplit_cache_slots: always enough for one
    step).  keep_device=False drops the device copies of Kp / Vp."""
    s = layer.shape
    if Hq is None:
        Hq = s.Hq
    shape = make_shape(s.B, s.S, Hq, s.Hkv, s.d, 1, s.kv_dtype)
    if n_slots is None:
        n_slots = cache_slots(shape, layer.cfg, budget)
    dev = layer.block_starts.device
    Kh = layer.Kp.cpu().pin_memory()
    Vh = layer.Vp.cpu().pin_memory()
    B, Hkv, _, P, d = layer.Kp.shape
    Kc = torch.zeros(B, Hkv, n_slots, P, d, dtype=layer.Kp.dtype, device=dev)
    Vc = torch.zeros_like(Kc)
    res = PagedLayer(shape, layer.cfg, layer.w10, layer.block_starts, layer.n_blocks, layer.page_first,
                     layer.page_block, layer.page_valid, layer.n_pages,
                     layer.Kp if keep_device else None, layer.Vp if keep_device else None, layer.digests)
    i32 = dict(dtype=torch.int32, device=dev)
    return OffloadedLayer(res, Kh, Vh, n_slots, torch.full((B, Hkv, n_slots), -1, **i32), Kc, Vc,
                          torch.zeros(B, Hkv, n_slots, 2, **i32), torch.zeros(B, Hkv, **i32),
                          torch.zeros(B, Hkv, 2, **i32), torch.zeros(B, **i32),
                          torch.zeros(worklist_bytes(shape, layer.cfg, budget), dtype=torch.uint8, device=dev))


def _host_ptr(t: torch.Tensor):
    if t.is_cuda or not t.is_pinned():
        raise DynsplitError("expected a pinned host tensor")
    return ctypes.c_void_p(t.data_ptr())


def reuse_plan(off: OffloadedLayer, worklist, Hq: Optional[int] = None, truncate: bool = True, reuse: bool = True,
               ws=None):
    """dynsplit_reuse_plan: Steps 1 and 3 against the cache's previous pages."""
    s = off.layer.shape
    Hq = Hq or s.Hq
    shape = make_shape(s.B, s.S, Hq, s.Hkv, s.d, 1, s.kv_dtype)
    if ws is None:
        ws = workspace(workspace_bytes(OP_REUSE, shape, off.layer.cfg), worklist.device, "reuse")
    c = off.c()
    _check(lib().dynsplit_reuse_plan(ctypes.byref(shape), ctypes.byref(off.layer.cfg), _ptr(worklist),
                                     int(truncate), int(reuse), ctypes.byref(c), _ptr(ws), ws.numel(), _stream()),
           "reuse_plan")


def fetch_pages(off: OffloadedLayer, Hq: Optional[int] = None, dense: bool = False) -> None:
    """dynsplit_fetch_pages: move the planned pages (dense: every page) host -> cache."""
    s = off.layer.shape
    Hq = Hq or s.Hq
    shape = make_shape(s.B, s.S, Hq, s.Hkv, s.d, 1, s.kv_dtype)
    c = off.c()
    _check(lib().dynsplit_fetch_pages(ctypes.byref(shape), ctypes.byref(off.layer.cfg), _host_ptr(off.Kh),
                                      _host_ptr(off.Vh), _ptr(off.layer.page_valid), _ptr(off.layer.n_pages),
                                      int(dense), ctypes.byref(c), _stream()), "fetch_pages")


def cache_view(off: OffloadedLayer) -> PagedLayer:
    """The cache as a PagedLayer (Kp = Kc, page stride n_slots) for dynsplit_decode_attn."""
    lay = off.layer
    cfg = Config.from_buffer_copy(lay.cfg)
    cfg.page_cap = off.n_slots
    return PagedLayer(lay.shape, cfg, lay.w10, lay.block_starts, lay.n_blocks, lay.page_first, lay.page_block,
                      lay.page_valid, lay.n_pages, off.Kc, off.Vc, lay.digests)


def decode_layer_offload(q, off: OffloadedLayer, budget: int, truncate: bool = True, reuse: bool = True,
                         scale: float = 0.0, out=None, ws=None):
    """dynsplit_decode_layer_offload: a5+a6 on the resident digests, the reuse
    plan, the move of the fresh pages from pinned host memory, a7+a8 over the
    cache.  out = (n_sel, marginal_block, marginal_keep, worklist, o, lse).
    -> (o, lse, Selection without scores / sel_blocks)."""
    shape = _decode_shape(q, off.layer)
    lay = off.layer
    if out is None:
        _, ns, mg, kp, wl = _sel_outputs(shape, lay.cfg, budget, q.device, want_blocks=False)
        o = torch.empty(shape.B, shape.Hq, shape.d, dtype=torch.float32, device=q.device)
        lse = torch.empty(shape.B, shape.Hq, dtype=torch.float32, device=q.device)
    else:
        ns, mg, kp, wl, o, lse = out
    if ws is None:
        ws = workspace(workspace_bytes(OP_DECODE_OFFLOAD, shape, lay.cfg, budget), q.device, "offload")
    c = off.c()
    _check(lib().dynsplit_decode_layer_offload(
        ctypes.byref(shape), ctypes.byref(lay.cfg), budget, _ptr(q), _ptr(lay.digests), _ptr(lay.block_starts),
        _ptr(lay.n_blocks), _ptr(lay.page_first), _ptr(lay.page_valid), _host_ptr(off.Kh), _host_ptr(off.Vh),
        int(truncate), int(reuse), ctypes.byref(c), ctypes.c_float(scale), _ptr(ns), _ptr(mg), _ptr(kp), _ptr(wl),
        _ptr(o), _ptr(lse), _ptr(ws), ws.numel(), _stream()), "decode_layer_offload")
    return o, lse, Selection(None, ns, mg, kp, wl, None)


def worklist_pages(worklist: torch.Tensor, shape: Shape):
    """Host-side reading of a worklist (tests and metrics): per (b, KV head)
    the page field of its entries, in entry order."""
    import numpy as np
    raw = worklist.cpu().numpy()
    nbh = shape.B * shape.Hkv
    max_wl = int(raw[:256].view(np.int32)[1])
    counts = raw[256:256 + 4 * nbh].view(np.int32).copy()
    off = 256 + ((4 * nbh + 255) // 256) * 256
    ent = raw[off: off + 16 * nbh * max_wl].reshape(max_wl, nbh, 16).transpose(1, 0, 2)
    return [ent[i, : counts[i], 0:4].copy().view(np.int32).ravel() for i in range(nbh)]
