"""Thin Python binding of libloza.so (include/loza.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch supplies
device memory, streams and (for sequence parallelism) the NCCL communicator.
There is no CPU or eager fallback: if the extension is missing this module
raises at import-use time.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# LOZA_LIB: development override (A/B builds of the same library, tools/build_variant.py); default in-tree .so
LIB_PATH = os.environ.get("LOZA_LIB") or os.path.join(_HERE, "libloza.so")

LOZA_F32, LOZA_BF16 = 0, 1
LOZA_WS_DECODE, LOZA_WS_FULL_DECODE, LOZA_WS_BLEND, LOZA_WS_SEQPAR, LOZA_WS_BACKWARD = 0, 1, 2, 3, 4
STATUS = {0: "LOZA_OK", 1: "LOZA_ERR_INVALID", 2: "LOZA_ERR_SHAPE", 3: "LOZA_ERR_UNSUPPORTED",
          4: "LOZA_ERR_CUDA", 5: "LOZA_ERR_NCCL"}

PAPER_PATTERN = (1, 7, 128)  # (s, l, b)
EXPORTS = ["ssa_prefill", "ssa_decode", "full_attn_ref", "loza_blend", "ssa_prefill_blend", "attention_backward",
           "ssa_prefill_mha", "ssa_ring_append",
           "ssa_decode_ring", "ssa_seqpar_prefill", "loza_seqpar_plan", "loza_seqpar_segments",
           "loza_seqpar_prefill_local", "loza_seqpar_prefill_loopback", "ssa_select_blocks", "loza_workspace_size", "loza_status_string",
           "loza_last_error", "loza_kernel_launches", "loza_num_sms", "loza_debug_force_kernel",
           "loza_workspace_init"]


class LozaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Pattern(ctypes.Structure):
    _fields_ = [("sink_blocks", ctypes.c_int32), ("local_blocks", ctypes.c_int32), ("block_size", ctypes.c_int32)]


class AttnArgs(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("n_q", ctypes.c_int32), ("heads", ctypes.c_int32),
                ("d_qk", ctypes.c_int32), ("d_v", ctypes.c_int32), ("n_kv", ctypes.c_int64),
                ("q_start", ctypes.c_int64), ("in_dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32),
                ("softmax_scale", ctypes.c_float), ("causal", ctypes.c_int32),
                ("q", ctypes.c_void_p), ("q_stride_b", ctypes.c_int64), ("q_stride_tok", ctypes.c_int64),
                ("q_stride_head", ctypes.c_int64),
                ("k", ctypes.c_void_p), ("k_stride_b", ctypes.c_int64), ("k_stride_tok", ctypes.c_int64),
                ("v", ctypes.c_void_p), ("v_stride_b", ctypes.c_int64), ("v_stride_tok", ctypes.c_int64),
                ("o", ctypes.c_void_p), ("o_stride_b", ctypes.c_int64), ("o_stride_tok", ctypes.c_int64),
                ("o_stride_head", ctypes.c_int64), ("lse", ctypes.c_void_p)]


class Xfer(ctypes.Structure):
    """loza_xfer_t: one transfer of the sequence-parallel exchange plan."""
    _fields_ = [("op", ctypes.c_int32), ("peer", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("tensor", ctypes.c_int32), ("src_row", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("row_elems", ctypes.c_int64), ("ws_offset", ctypes.c_int64)]


XFER_BCAST, XFER_SEND, XFER_RECV = 0, 1, 2

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(there is no fallback path)")
        L = ctypes.CDLL(LIB_PATH)
        P, S, V, I32, I64, SZ = ctypes.POINTER, ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, \
            ctypes.c_size_t
        L.ssa_prefill.argtypes = [P(AttnArgs), Pattern, V]
        L.ssa_decode.argtypes = [P(AttnArgs), V, Pattern, V, SZ, V]
        L.full_attn_ref.argtypes = [P(AttnArgs), V, V, SZ, V]
        L.loza_blend.argtypes = [V, V, V, V, V, V, I64, S, V, V, SZ, V]
        L.ssa_prefill_blend.argtypes = [P(AttnArgs), Pattern, V, V, V, V, V, V, SZ, V]
        L.ssa_ring_append.argtypes = [V, I64, I64, I32, V, Pattern, V, I64, I64, I32, I32, S, V]
        L.attention_backward.argtypes = [P(AttnArgs), I32, Pattern, V, V, V, V, V, SZ, V]
        L.ssa_decode_ring.argtypes = [P(AttnArgs), V, Pattern, V]
        L.ssa_prefill_mha.argtypes = [P(AttnArgs), I64, I64, I32, Pattern, V]
        L.ssa_seqpar_prefill.argtypes = [P(AttnArgs), Pattern, V, I32, I32, V, SZ, V]
        L.loza_seqpar_prefill_local.argtypes = [P(AttnArgs), Pattern, I32, I32, V, V, V, V, V, SZ, V]
        L.loza_seqpar_prefill_loopback.argtypes = [P(AttnArgs), Pattern, V, I32, I32, V, V, V, V, V, SZ, V]
        L.loza_seqpar_plan.argtypes = [P(AttnArgs), Pattern, I32, I32, P(Xfer), I32]
        L.loza_seqpar_plan.restype = I32
        L.loza_seqpar_segments.argtypes = [P(AttnArgs), Pattern, I32, I32, P(I64)]
        L.loza_seqpar_segments.restype = I32
        L.ssa_select_blocks.argtypes = [I64, I64, Pattern, I32, V, V, V]
        L.loza_workspace_size.argtypes = [I32, P(AttnArgs), Pattern, I32]
        L.loza_workspace_size.restype = SZ
        L.loza_status_string.restype = ctypes.c_char_p
        L.loza_last_error.restype = ctypes.c_char_p
        L.loza_kernel_launches.restype = ctypes.c_uint64
        L.loza_num_sms.restype = I32
        L.loza_debug_force_kernel.argtypes = [ctypes.c_char_p, I32]
        L.loza_debug_force_kernel.restype = I32
        L.loza_workspace_init.argtypes = [I32, P(AttnArgs), Pattern, I32, V, SZ, V]
        L.loza_workspace_init.restype = S
        for fn in ("ssa_prefill", "ssa_decode", "full_attn_ref", "loza_blend", "ssa_seqpar_prefill",
                   "loza_seqpar_prefill_local", "loza_seqpar_prefill_loopback", "ssa_select_blocks"):
            getattr(L, fn).restype = S
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise LozaError(rc, lib().loza_last_error().decode())


def kernel_launches() -> int:
    return int(lib().loza_kernel_launches())


def force_kernel(family: str, variant: int) -> None:
    """Test hook (loza_debug_force_kernel): family "decode" (0 auto, 1 pair-cooperative, 2 key-split pair) or
    "backward" (0 auto, 1 FFMA, 2 warp-MMA keys and rows, 3 tcgen05 keys + warp-MMA dQ)."""
    if lib().loza_debug_force_kernel(family.encode(), int(variant)) != 0:
        raise ValueError(f"unknown kernel override {family}={variant}")


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return LOZA_BF16
    if t.dtype == torch.float32:
        return LOZA_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _pattern(pattern) -> Pattern:
    s, l, b = pattern
    return Pattern(int(s), int(l), int(b))


def _q4(q):  # [B,n,H,d] view
    return q if q.dim() == 4 else q.unsqueeze(0)


def _kv3(k):  # [B,n,d] view
    return k if k.dim() == 3 else k.unsqueeze(0)


def make_args(q, k, v, o, *, scale, causal=True, q_start=0, n_kv=None, lse=None) -> AttnArgs:
    """q [B,n_q,H,dqk]; k [B,n_kv,dqk]; v [B,n_kv,dv] (for MLA pass v = k[..., :512]); o [B,n_q,H,dv]."""
    q4, o4 = _q4(q), _q4(o)
    k3, v3 = _kv3(k), _kv3(v)
    for t in (q4, k3, v3, o4):
        if not t.is_cuda:
            raise ValueError("all tensors must be CUDA tensors (no CPU path)")
        if t.stride(-1) != 1:
            raise ValueError("innermost dimension must be contiguous")
    B, n_q, H, dqk = q4.shape
    dv = v3.shape[-1]
    a = AttnArgs()
    a.batch, a.n_q, a.heads, a.d_qk, a.d_v = B, n_q, H, dqk, dv
    a.n_kv = k3.shape[1] if n_kv is None else n_kv
    a.q_start = q_start
    a.in_dtype, a.out_dtype = _dt(q4), _dt(o4)
    a.softmax_scale = float(scale)
    a.causal = 1 if causal else 0
    a.q, a.q_stride_b, a.q_stride_tok, a.q_stride_head = q4.data_ptr(), q4.stride(0), q4.stride(1), q4.stride(2)
    a.k, a.k_stride_b, a.k_stride_tok = k3.data_ptr(), k3.stride(0), k3.stride(1)
    a.v, a.v_stride_b, a.v_stride_tok = v3.data_ptr(), v3.stride(0), v3.stride(1)
    a.o, a.o_stride_b, a.o_stride_tok, a.o_stride_head = o4.data_ptr(), o4.stride(0), o4.stride(1), o4.stride(2)
    a.lse = lse.data_ptr() if lse is not None else None
    return a


def _split_kv(k, v, d_v):
    if v is None:  # MLA: V = first d_v columns of the latent KV row
        v = k[..., :d_v]
    return k, v


def _alloc_out(q, dv, out_dtype):
    q4 = _q4(q)
    shape = (*q4.shape[:3], dv)
    o = torch.empty(shape, dtype=out_dtype or q4.dtype, device=q4.device)
    return o if q.dim() == 4 else o[0]


def default_scale(d_qk: int) -> float:
    """1/sqrt(192) for absorbed MLA (128 nope + 64 RoPE per head, DESIGN R1), else 1/sqrt(d)."""
    return 1.0 / math.sqrt(192.0) if d_qk == 576 else 1.0 / math.sqrt(d_qk)


def ssa_prefill(q, k, v=None, pattern=PAPER_PATTERN, scale=None, *, d_v=512, out=None, lse=None, q_start=0,
                out_dtype=None, stream=None):
    """SSA prefill, Eq. 4. Returns O [.., n_q, H, d_v]."""
    k, v = _split_kv(k, v, d_v)
    scale = default_scale(q.shape[-1]) if scale is None else scale
    o = out if out is not None else _alloc_out(q, v.shape[-1], out_dtype)
    a = make_args(q, k, v, o, scale=scale, q_start=q_start, lse=lse)
    _check(lib().ssa_prefill(ctypes.byref(a), _pattern(pattern), _stream(stream)))
    return o


def ssa_prefill_blend(q, k, o_full, alpha, d_o_hat=None, v=None, pattern=PAPER_PATTERN, scale=None, *, d_v=512,
                      out=None, q_start=0, status=None, stream=None):
    """Fused calibration forward (Eq. 3 with O' = SSA prefill, never stored): returns (o_hat, d_alpha or None).
    alpha: 1-element fp32 CUDA tensor; o_full / d_o_hat: bf16, o's shape [.., n_q, H, d_v]."""
    k, v = _split_kv(k, v, d_v)
    scale = default_scale(q.shape[-1]) if scale is None else scale
    o = out if out is not None else _alloc_out(q, v.shape[-1], torch.bfloat16)
    assert o_full.shape == o.shape and o_full.dtype == torch.bfloat16 and o_full.is_contiguous()
    assert alpha.dtype == torch.float32 and alpha.is_cuda
    a = make_args(q, k, v, o, scale=scale, q_start=q_start)
    d_alpha = None
    if d_o_hat is not None:
        assert d_o_hat.shape == o.shape and d_o_hat.dtype == torch.bfloat16 and d_o_hat.is_contiguous()
        d_alpha = torch.empty(1, dtype=torch.float64, device=q.device)
    need, ws = _blend_workspace(stream)
    V = ctypes.c_void_p
    _check(lib().ssa_prefill_blend(ctypes.byref(a), _pattern(pattern), V(o_full.data_ptr()), V(alpha.data_ptr()),
                                   V(d_o_hat.data_ptr() if d_o_hat is not None else 0),
                                   V(d_alpha.data_ptr() if d_alpha is not None else 0),
                                   V(status.data_ptr() if status is not None else 0), V(ws.data_ptr()), need,
                                   _stream(stream)))
    return o, d_alpha


def attention_backward(q, k, o, lse, d_o, v=None, pattern=PAPER_PATTERN, scale=None, *, d_v=512, causal=True,
                       q_start=0, stream=None):
    """Gradients of SSA (pattern) or full attention (pattern=None) for dL/dO = d_o, given the forward's
    q, k (v: default MLA slice of k), o and lse [B,H,n_q]. Returns fp32 (d_q [B,n_q,H,dqk], d_k [B,n_kv,dqk],
    d_v [B,n_kv,dv]); for the MLA cache the gradient is d_k + [d_v, 0]."""
    k, v = _split_kv(k, v, d_v)
    scale = default_scale(q.shape[-1]) if scale is None else scale
    a = make_args(q, k, v, o, scale=scale, causal=causal, q_start=q_start, lse=lse)
    o4 = _q4(o)
    if d_o.dtype != o.dtype or d_o.numel() != o4.numel():
        raise ValueError(f"d_o must match o (dtype {o.dtype}, {tuple(o4.shape)}); got {d_o.dtype}, {tuple(d_o.shape)}")
    do4 = d_o.reshape(o4.shape)
    if do4.stride() != o4.stride():
        raise ValueError(f"d_o must have o's layout: strides {o4.stride()} vs {do4.stride()}")
    B, n_q, H, dqk = _q4(q).shape
    n_kv, dv = _kv3(k).shape[1], v.shape[-1]
    dq = torch.empty((B, n_q, H, dqk), dtype=torch.float32, device=q.device)
    dk = torch.empty((B, n_kv, dqk), dtype=torch.float32, device=q.device)
    dvv = torch.empty((B, n_kv, dv), dtype=torch.float32, device=q.device)
    pat = pattern if pattern is not None else (0, 1, 1)
    need = lib().loza_workspace_size(LOZA_WS_BACKWARD, ctypes.byref(a), _pattern(pat), 1)
    with torch.cuda.stream(torch.cuda.current_stream() if stream is None else stream):  # freed after the launch
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device=q.device)
    V = ctypes.c_void_p
    _check(lib().attention_backward(ctypes.byref(a), 1 if pattern is not None else 0, _pattern(pat),
                                    V(do4.data_ptr()), V(dq.data_ptr()), V(dk.data_ptr()), V(dvv.data_ptr()),
                                    V(ws.data_ptr()), need, _stream(stream)))
    return dq, dk, dvv


def ssa_prefill_mha(q, k, v, pattern=PAPER_PATTERN, scale=None, *, sparse=True, causal=True, out=None, lse=None,
                    q_start=0, out_dtype=None, stream=None):
    """Non-absorbed (MHA-form) SSA prefill: q [B,n_q,H,192], k [B,n_kv,H,192], v [B,n_kv,H,128]
    (per-head K/V; any strides with a contiguous innermost dim). sparse=False: the full-attention comparator.
    Returns O [B,n_q,H,128]."""
    for t in (q, k, v):
        if t.dim() != 4 or not t.is_cuda or t.stride(-1) != 1:
            raise ValueError("q, k, v must be 4-D CUDA tensors [B, n, H, d] with a contiguous last dim")
    B, n_q, H, dqk = q.shape
    scale = 1.0 / math.sqrt(dqk) if scale is None else scale
    o = out if out is not None else torch.empty((B, n_q, H, v.shape[-1]), dtype=out_dtype or q.dtype,
                                                device=q.device)
    a = AttnArgs()
    a.batch, a.n_q, a.heads, a.d_qk, a.d_v = B, n_q, H, dqk, v.shape[-1]
    a.n_kv, a.q_start = k.shape[1], q_start
    a.in_dtype, a.out_dtype = _dt(q), _dt(o)
    a.softmax_scale, a.causal = float(scale), 1 if causal else 0
    a.q, a.q_stride_b, a.q_stride_tok, a.q_stride_head = q.data_ptr(), q.stride(0), q.stride(1), q.stride(2)
    a.k, a.k_stride_b, a.k_stride_tok = k.data_ptr(), k.stride(0), k.stride(1)
    a.v, a.v_stride_b, a.v_stride_tok = v.data_ptr(), v.stride(0), v.stride(1)
    a.o, a.o_stride_b, a.o_stride_tok, a.o_stride_head = o.data_ptr(), o.stride(0), o.stride(1), o.stride(2)
    a.lse = lse.data_ptr() if lse is not None else None
    _check(lib().ssa_prefill_mha(ctypes.byref(a), k.stride(2), v.stride(2), 1 if sparse else 0, _pattern(pattern),
                                 _stream(stream)))
    return o


def ring_rows(pattern=PAPER_PATTERN) -> int:
    s, l, b = pattern
    return (s + l) * b


def ssa_ring_append(cache, rows, pos0, pattern=PAPER_PATTERN, stream=None):
    """Append rows [B, m, d] at absolute positions pos0[b] .. (int32 CUDA tensor [B]) to the ring cache
    [B, (s+l)*b, d] (bounded SSA KV cache, block-boundary eviction)."""
    assert cache.dim() == 3 and rows.dim() == 3 and rows.dtype == cache.dtype and rows.shape[-1] == cache.shape[-1]
    assert cache.shape[1] == ring_rows(pattern) and pos0.dtype == torch.int32 and pos0.is_cuda
    V = ctypes.c_void_p
    _check(lib().ssa_ring_append(V(rows.data_ptr()), rows.stride(0), rows.stride(1), rows.shape[1],
                                 V(pos0.data_ptr()), _pattern(pattern), V(cache.data_ptr()), cache.stride(0),
                                 cache.stride(1), rows.shape[0], rows.shape[-1], _dt(rows), _stream(stream)))
    return cache


def ssa_decode_ring(q, cache, seq_lens, v=None, pattern=PAPER_PATTERN, scale=None, *, d_v=512, out=None, lse=None,
                    out_dtype=None, stream=None):
    """SSA decode over the bounded ring cache [B, (s+l)*b, d_qk]; seq_lens: absolute lengths (int32 CUDA [B])."""
    q4 = q if q.dim() == 4 else q.unsqueeze(1)
    k, v = _split_kv(cache, v, d_v)
    scale = default_scale(q4.shape[-1]) if scale is None else scale
    o = out if out is not None else torch.empty((*q4.shape[:3], v.shape[-1]), dtype=out_dtype or q4.dtype,
                                                device=q4.device)
    o4 = o if o.dim() == 4 else o.unsqueeze(1)
    a = make_args(q4, k, v, o4, scale=scale, lse=lse)
    assert seq_lens.dtype == torch.int32 and seq_lens.is_cuda
    _check(lib().ssa_decode_ring(ctypes.byref(a), ctypes.c_void_p(seq_lens.data_ptr()), _pattern(pattern),
                                 _stream(stream)))
    return o if q.dim() == 4 else o4[:, 0]


_decode_ws_cache = {}


def _decode_ws(which, a, pattern, ws, stream):
    """Decode workspace (include/loza.h): a status word, then (flattened split-KV kernel) per-sequence counters and
    partials. It must start zeroed (loza_workspace_init) and every call leaves the counters at zero, so one buffer
    is initialised once per (device, stream) and reused; concurrent streams get their own."""
    need = lib().loza_workspace_size(which, ctypes.byref(a), _pattern(pattern), 1)
    if need == 0:
        return None, 0
    if ws is None or ws.numel() < need:
        s = torch.cuda.current_stream() if stream is None else stream
        key = (s.device.index, s.cuda_stream, which)
        ws = _decode_ws_cache.get(key)
        if ws is None or ws.numel() < need:
            with torch.cuda.stream(s):
                ws = torch.empty(need, dtype=torch.uint8, device=s.device)
            _check(lib().loza_workspace_init(which, ctypes.byref(a), _pattern(pattern), 1,
                                             ctypes.c_void_p(ws.data_ptr()), need, ctypes.c_void_p(s.cuda_stream)))
            _decode_ws_cache[key] = ws
    return ws, need


def decode_status(ws) -> int:
    """The status word of a decode workspace: LOZA_ERR_SHAPE (2) once some seq_len was outside [1, n_kv] (the
    kernels clamp it and continue), else 0. Synchronises with the device."""
    return int(ws[:4].view(torch.int32).item())


def decode_status_reset(ws, stream=None):
    ws[:4].zero_()


def ssa_decode(q, cache, seq_lens, v=None, pattern=PAPER_PATTERN, scale=None, *, d_v=512, out=None, lse=None,
               ws=None, out_dtype=None, stream=None):
    """SSA decode: q [B,1,H,dqk] (or [B,H,dqk]), cache [B,T_cap,dqk], seq_lens int32 [B] on the device."""
    q4 = q if q.dim() == 4 else q.unsqueeze(1)
    k, v = _split_kv(cache, v, d_v)
    scale = default_scale(q4.shape[-1]) if scale is None else scale
    o = out if out is not None else torch.empty((*q4.shape[:3], v.shape[-1]), dtype=out_dtype or q4.dtype,
                                                device=q4.device)
    o4 = o if o.dim() == 4 else o.unsqueeze(1)
    a = make_args(q4, k, v, o4, scale=scale, lse=lse)
    assert seq_lens.dtype == torch.int32 and seq_lens.is_cuda
    w, need = _decode_ws(LOZA_WS_DECODE, a, pattern, ws, stream)
    _check(lib().ssa_decode(ctypes.byref(a), ctypes.c_void_p(seq_lens.data_ptr()), _pattern(pattern),
                            ctypes.c_void_p(w.data_ptr() if w is not None else 0), need, _stream(stream)))
    return o if q.dim() == 4 else o4[:, 0]


def full_attn_ref(q, k, v=None, scale=None, *, seq_lens=None, causal=True, d_v=512, out=None, lse=None, q_start=0,
                  ws=None, out_dtype=None, stream=None):
    """Full attention comparator, Eq. 1. Prefill (seq_lens None) or decode (q [B,1,H,d], cache, seq_lens)."""
    k, v = _split_kv(k, v, d_v)
    scale = default_scale(q.shape[-1]) if scale is None else scale
    if seq_lens is None:
        o = out if out is not None else _alloc_out(q, v.shape[-1], out_dtype)
        a = make_args(q, k, v, o, scale=scale, causal=causal, q_start=q_start, lse=lse)
        _check(lib().full_attn_ref(ctypes.byref(a), None, None, 0, _stream(stream)))
        return o
    q4 = q if q.dim() == 4 else q.unsqueeze(1)
    o = out if out is not None else torch.empty((*q4.shape[:3], v.shape[-1]), dtype=out_dtype or q4.dtype,
                                                device=q4.device)
    o4 = o if o.dim() == 4 else o.unsqueeze(1)
    a = make_args(q4, k, v, o4, scale=scale, causal=causal, lse=lse)
    w, need = _decode_ws(LOZA_WS_FULL_DECODE, a, (0, 1, 1), ws, stream)
    _check(lib().full_attn_ref(ctypes.byref(a), ctypes.c_void_p(seq_lens.data_ptr()),
                               ctypes.c_void_p(w.data_ptr() if w is not None else 0), need, _stream(stream)))
    return o if q.dim() == 4 else o4[:, 0]


_blend_ws = {}


def _blend_workspace(stream):
    """Per-CTA d_alpha partials (written and reduced inside one call): one buffer per (device, stream)."""
    need = lib().loza_workspace_size(LOZA_WS_BLEND, None, Pattern(0, 1, 1), 1)
    s = torch.cuda.current_stream() if stream is None else stream
    key = (s.device.index, s.cuda_stream)
    ws = _blend_ws.get(key)
    if ws is None:
        with torch.cuda.stream(s):
            ws = _blend_ws[key] = torch.empty(need, dtype=torch.uint8, device=s.device)
    return need, ws


def loza_blend(o_full, o_sparse, alpha, d_o_hat=None, *, out=None, d_alpha=None, status=None, want_out=True,
               stream=None):
    """Eq. 3 blend. alpha: 1-element fp32 CUDA tensor. Returns (o_hat or None, d_alpha fp64 tensor or None)."""
    assert o_full.shape == o_sparse.shape and o_full.dtype == o_sparse.dtype
    assert o_full.is_contiguous() and o_sparse.is_contiguous()
    assert alpha.dtype == torch.float32 and alpha.is_cuda
    dev = o_full.device
    o_hat = None
    if want_out:
        o_hat = out if out is not None else torch.empty_like(o_full)
    if d_o_hat is not None:
        assert d_o_hat.shape == o_full.shape and d_o_hat.dtype == o_full.dtype and d_o_hat.is_contiguous()
        if d_alpha is None:
            d_alpha = torch.empty(1, dtype=torch.float64, device=dev)
    need, ws = _blend_workspace(stream)
    V = ctypes.c_void_p
    _check(lib().loza_blend(V(o_full.data_ptr()), V(o_sparse.data_ptr()), V(alpha.data_ptr()),
                            V(o_hat.data_ptr() if o_hat is not None else 0),
                            V(d_o_hat.data_ptr() if d_o_hat is not None else 0),
                            V(d_alpha.data_ptr() if d_o_hat is not None else 0), o_full.numel(), _dt(o_full),
                            V(status.data_ptr() if status is not None else 0), V(ws.data_ptr()), need,
                            _stream(stream)))
    return o_hat, (d_alpha if d_o_hat is not None else None)


def ssa_select_blocks(n_q: int, q_start: int = 0, pattern=PAPER_PATTERN, stream=None):
    s, l, b = pattern
    nqb = (n_q + b - 1) // b
    idx = torch.empty((max(nqb, 1), s + l), dtype=torch.int32, device="cuda")
    cnt = torch.empty(max(nqb, 1), dtype=torch.int32, device="cuda")
    _check(lib().ssa_select_blocks(n_q, q_start, _pattern(pattern), 1, ctypes.c_void_p(idx.data_ptr()),
                                   ctypes.c_void_p(cnt.data_ptr()), _stream(stream)))
    return idx[:nqb], cnt[:nqb]


def seqpar_ws_bytes(q_shard, k_shard, v_shard, pattern, world) -> int:
    o = torch.empty(0, device=q_shard.device, dtype=q_shard.dtype)
    a = make_args(q_shard, k_shard, v_shard, q_shard[..., :v_shard.shape[-1]], scale=1.0)
    del o
    return int(lib().loza_workspace_size(LOZA_WS_SEQPAR, ctypes.byref(a), _pattern(pattern), world))


def ssa_seqpar_prefill(q_shard, k_shard, v=None, pattern=PAPER_PATTERN, scale=None, *, rank: int, world: int,
                       comm_ptr: int = 0, d_v=512, out=None, lse=None, ws=None, out_dtype=None, stream=None):
    """Sequence-parallel SSA prefill of this rank's shard (see include/loza.h). comm_ptr: ncclComm_t as int
    (e.g. ProcessGroupNCCL._comm_ptr()), 0 allowed for world == 1."""
    k_shard, v = _split_kv(k_shard, v, d_v)
    scale = default_scale(q_shard.shape[-1]) if scale is None else scale
    n_local = _q4(q_shard).shape[1]
    o = out if out is not None else _alloc_out(q_shard, v.shape[-1], out_dtype)
    a = make_args(q_shard, k_shard, v, o, scale=scale, q_start=rank * n_local, lse=lse)
    need = int(lib().loza_workspace_size(LOZA_WS_SEQPAR, ctypes.byref(a), _pattern(pattern), world))
    if ws is None or ws.numel() < need:
        with torch.cuda.stream(torch.cuda.current_stream() if stream is None else stream):
            ws = torch.empty(max(need, 1), dtype=torch.uint8, device=q_shard.device)
    _check(lib().ssa_seqpar_prefill(ctypes.byref(a), _pattern(pattern), ctypes.c_void_p(comm_ptr), rank, world,
                                    ctypes.c_void_p(ws.data_ptr()), need, _stream(stream)))
    return o


def ssa_seqpar_prefill_local(q_shard, k_shard, v=None, pattern=PAPER_PATTERN, scale=None, *, rank: int, world: int,
                             rank0_k=None, rank0_v=None, prev_k=None, prev_v=None, d_v=512, out=None, lse=None,
                             out_dtype=None, stream=None):
    """Virtual-rank test hook: the exchange is done by device copies from the other shards on this GPU."""
    k_shard, v = _split_kv(k_shard, v, d_v)
    scale = default_scale(q_shard.shape[-1]) if scale is None else scale
    n_local = _q4(q_shard).shape[1]
    o = out if out is not None else _alloc_out(q_shard, v.shape[-1], out_dtype)
    a = make_args(q_shard, k_shard, v, o, scale=scale, q_start=rank * n_local, lse=lse)
    need = int(lib().loza_workspace_size(LOZA_WS_SEQPAR, ctypes.byref(a), _pattern(pattern), world))
    with torch.cuda.stream(torch.cuda.current_stream() if stream is None else stream):
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device=q_shard.device)
    V = ctypes.c_void_p

    def ptr(t):
        return V(t.data_ptr() if t is not None else 0)
    if v.data_ptr() == k_shard.data_ptr():
        rank0_v = rank0_k if rank0_v is None else rank0_v
        prev_v = prev_k if prev_v is None else prev_v
    _check(lib().loza_seqpar_prefill_local(ctypes.byref(a), _pattern(pattern), rank, world, ptr(rank0_k),
                                           ptr(rank0_v), ptr(prev_k), ptr(prev_v), V(ws.data_ptr()), need,
                                           _stream(stream)))
    return o


def seqpar_host_args(n_local: int, rank: int, *, batch=1, heads=64, d_qk=576, d_v=512, alias=True,
                     dtype=LOZA_BF16) -> AttnArgs:
    """AttnArgs describing rank `rank`'s shard for the host-only plan queries (no tensors: the plan and the
    segments depend on shapes, strides and whether v aliases k only)."""
    a = AttnArgs()
    a.batch, a.n_q, a.heads, a.d_qk, a.d_v = batch, n_local, heads, d_qk, d_v
    a.n_kv, a.q_start = n_local, rank * n_local
    a.in_dtype = a.out_dtype = dtype
    a.softmax_scale, a.causal = 1.0, 1
    a.q_stride_b, a.q_stride_tok, a.q_stride_head = n_local * heads * d_qk, heads * d_qk, d_qk
    a.k = 4096  # stand-in addresses: only k == v (MLA aliasing) matters to the plan
    a.k_stride_b, a.k_stride_tok = n_local * d_qk, d_qk
    a.v = a.k if alias else 8192
    a.v_stride_b, a.v_stride_tok = (n_local * d_qk, d_qk) if alias else (n_local * d_v, d_v)
    a.o_stride_b, a.o_stride_tok, a.o_stride_head = n_local * heads * d_v, heads * d_v, d_v
    return a


def seqpar_plan(a: AttnArgs, pattern, rank: int, world: int):
    """The exchange plan (list of dicts, issue order) ssa_seqpar_prefill executes for this rank."""
    n = lib().loza_seqpar_plan(ctypes.byref(a), _pattern(pattern), rank, world, None, 0)
    if n < 0:
        _check(-n)
    buf = (Xfer * max(n, 1))()
    lib().loza_seqpar_plan(ctypes.byref(a), _pattern(pattern), rank, world, buf, n)
    return [{f: getattr(buf[i], f) for f, _ in Xfer._fields_} for i in range(n)]


def seqpar_segments(a: AttnArgs, pattern, rank: int, world: int):
    """Segments of the KV view after the exchange: dicts with pos_begin, pos_end, k_off, v_off (ws byte offsets
    for batch 0, -1 = the shard's own rows), k_sb, v_sb (batch strides in bytes)."""
    out = (ctypes.c_int64 * 18)()
    n = lib().loza_seqpar_segments(ctypes.byref(a), _pattern(pattern), rank, world, out)
    if n < 0:
        _check(-n)
    keys = ("pos_begin", "pos_end", "k_off", "v_off", "k_sb", "v_sb")
    return [{k: out[6 * i + j] for j, k in enumerate(keys)} for i in range(n)]


def ssa_seqpar_prefill_loopback(q_shard, k_shard, v=None, pattern=PAPER_PATTERN, scale=None, *, rank: int,
                                world: int, comm_ptr: int, rank0_k=None, rank0_v=None, prev_k=None, prev_v=None,
                                d_v=512, out=None, lse=None, out_dtype=None, stream=None):
    """Test hook: the exchange through NCCL on a one-rank communicator (comm_ptr), virtual ranks on one GPU."""
    k_shard, v = _split_kv(k_shard, v, d_v)
    scale = default_scale(q_shard.shape[-1]) if scale is None else scale
    n_local = _q4(q_shard).shape[1]
    o = out if out is not None else _alloc_out(q_shard, v.shape[-1], out_dtype)
    a = make_args(q_shard, k_shard, v, o, scale=scale, q_start=rank * n_local, lse=lse)
    need = int(lib().loza_workspace_size(LOZA_WS_SEQPAR, ctypes.byref(a), _pattern(pattern), world))
    s = torch.cuda.current_stream() if stream is None else stream
    with torch.cuda.stream(s):
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device=q_shard.device)
    V = ctypes.c_void_p

    def ptr(t):
        return V(t.data_ptr() if t is not None else 0)
    if v.data_ptr() == k_shard.data_ptr():
        rank0_v = rank0_k if rank0_v is None else rank0_v
        prev_v = prev_k if prev_v is None else prev_v
    _check(lib().loza_seqpar_prefill_loopback(ctypes.byref(a), _pattern(pattern), V(comm_ptr), rank, world,
                                              ptr(rank0_k), ptr(rank0_v), ptr(prev_k), ptr(prev_v),
                                              V(ws.data_ptr()), need, _stream(stream)))
    return o
