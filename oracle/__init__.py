"""fp64 CPU oracle for the LoZA / SSA hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. It shares no code with the CUDA path
(paper_2512_23966_b200/) and never imports it; the CUDA path never imports it.

The arithmetic lives in ``loza_oracle.c`` (C99 + OpenMP, fp64), each function
citing the passage it follows (Eq. 1, 3, 4 of PAPER.md and the SPEC.md:121 mask).
This module only marshals numpy arrays. Parity pins: tests/test_oracle_pins.py.
Parity unpinned: none of the functions (see DESIGN.md §"Oracle and pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "loza_oracle.c")
LIB_PATH = os.path.join(_HERE, "liblozaoracle.so")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64, _i32, _dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_double


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared", SRC, "-o", LIB_PATH, "-lm"],
                       check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.loza_oracle_mask_row.restype = None
        L.loza_oracle_mask_row.argtypes = [_i64, _i64, _i32, _i32, _i32, _i32, _i32, _u8p]
        L.loza_oracle_allowed_keys.restype = _i64
        L.loza_oracle_allowed_keys.argtypes = [_i64, _i64, _i32, _i32, _i32, _i32, _i32, _i64p]
        L.loza_oracle_select_blocks.restype = ctypes.c_int
        L.loza_oracle_select_blocks.argtypes = [_i64, _i64, _i64, _i32, _i32, _i32, _i32, _i64p, _i64, _i32,
                                                _i32p, _i32p]
        L.loza_oracle_attend.restype = None
        L.loza_oracle_attend.argtypes = [_f32p, _i64, _i64, _f32p, _i64, _f32p, _i64, _i64, _i32, _i32, _dbl,
                                         _f64p, _f64p]
        L.loza_oracle_attention_rows.restype = None
        L.loza_oracle_attention_rows.argtypes = [_f32p, _i64p, _i64, _i64, _f32p, _i64, _f32p, _i64, _i64,
                                                 _i32, _i32, _dbl, _i32, _i32, _i32, _i32, _i32, _f64p, _f64p]
        L.loza_oracle_blend.restype = None
        L.loza_oracle_blend.argtypes = [_f32p, _f32p, _dbl, ctypes.c_void_p, _i64, ctypes.c_void_p,
                                        ctypes.c_void_p]
        L.loza_oracle_attention_backward.restype = None
        L.loza_oracle_attention_backward.argtypes = [_f32p, _i64p, _i64, _i64, _f32p, _i64, _f32p, _i64, _f32p,
                                                     _i64, _i64, _i32, _i32, _dbl, _i32, _i32, _i32, _i32, _i32,
                                                     _f64p, _f64p, _f64p]
        L.loza_oracle_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def num_threads() -> int:
    return lib().loza_oracle_num_threads()


def _c32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def mask_row(p: int, n_kv: int, s: int, l: int, b: int, sparse: bool = True, causal: bool = True) -> np.ndarray:
    out = np.empty(max(n_kv, 1), dtype=np.uint8)
    lib().loza_oracle_mask_row(p, n_kv, s, l, b, int(sparse), int(causal), out)
    return out[:n_kv]


def allowed_keys(p: int, n_kv: int, s: int, l: int, b: int, sparse: bool = True,
                 causal: bool = True) -> np.ndarray:
    out = np.empty(max(n_kv, 1), dtype=np.int64)
    c = lib().loza_oracle_allowed_keys(p, n_kv, s, l, b, int(sparse), int(causal), out)
    return out[:c].copy()


def select_blocks(n_q: int, q_start: int, n_kv: int, s: int, l: int, b: int, causal: bool = True,
                  qb_list=None, max_sel: int | None = None):
    """Oracle block selection for local query blocks ``qb_list`` (default: all)."""
    n_qb = (n_q + b - 1) // b
    qbs = np.arange(n_qb, dtype=np.int64) if qb_list is None else np.ascontiguousarray(qb_list, dtype=np.int64)
    if max_sel is None:
        max_sel = s + l
    idx = np.empty((max(len(qbs), 1), max_sel), dtype=np.int32)
    cnt = np.empty(max(len(qbs), 1), dtype=np.int32)
    rc = lib().loza_oracle_select_blocks(n_q, q_start, n_kv, s, l, b, int(causal), qbs, len(qbs), max_sel,
                                         idx, cnt)
    if rc != 0:
        raise ValueError("a query block selected more than max_sel key blocks")
    return idx[:len(qbs)], cnt[:len(qbs)]


def attend(q, k, v, scale: float):
    """softmax(scale q k^T) v over exactly the given key rows. q [R,dqk], k [nk,dqk], v [nk,dv]."""
    q, k, v = _c32(q), _c32(k), _c32(v)
    R, dqk = q.shape
    nk, dv = v.shape
    o = np.empty((R, dv), dtype=np.float64)
    lse = np.empty(max(R, 1), dtype=np.float64)
    lib().loza_oracle_attend(q, R, dqk, k, k.shape[1], v, dv, nk, dqk, dv, float(scale), o, lse)
    return o, lse[:R]


def attention_rows(q_rows, pos, k, v, scale: float, s: int = 1, l: int = 7, b: int = 128,
                   sparse: bool = True, causal: bool = True):
    """Rows of O / LSE for queries q_rows [R,dqk] at absolute positions pos [R] against k [n_kv,dqk],
    v [n_kv,dv] (v may be a column slice of the latent KV: it is copied contiguous)."""
    q_rows, k, v = _c32(q_rows), _c32(k), _c32(v)
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    R, dqk = q_rows.shape
    n_kv, dv = v.shape
    assert k.shape[0] == n_kv and len(pos) == R
    o = np.empty((R, dv), dtype=np.float64)
    lse = np.empty(max(R, 1), dtype=np.float64)
    lib().loza_oracle_attention_rows(q_rows, pos, R, dqk, k, k.shape[1], v, dv, n_kv, dqk, dv, float(scale),
                                     s, l, b, int(sparse), int(causal), o, lse)
    return o, lse[:R]


def attention_backward(q_rows, pos, k, v, do_rows, scale: float, s: int = 1, l: int = 7, b: int = 128,
                       sparse: bool = True, causal: bool = True):
    """Backward of attention_rows for the loss with dL/dO = do_rows: returns (dq [R,dqk], dk [n_kv,dqk],
    dv [n_kv,dv]) in fp64."""
    q_rows, k, v, do_rows = _c32(q_rows), _c32(k), _c32(v), _c32(do_rows)
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    R, dqk = q_rows.shape
    n_kv, dv = v.shape
    assert k.shape[0] == n_kv and len(pos) == R and do_rows.shape == (R, dv)
    dq = np.empty((max(R, 1), dqk), dtype=np.float64)
    dk = np.empty((max(n_kv, 1), dqk), dtype=np.float64)
    dvo = np.empty((max(n_kv, 1), dv), dtype=np.float64)
    lib().loza_oracle_attention_backward(q_rows, pos, R, dqk, k, k.shape[1], v, dv, do_rows, dv, n_kv, dqk, dv,
                                         float(scale), s, l, b, int(sparse), int(causal), dq, dk, dvo)
    return dq[:R], dk[:n_kv], dvo[:n_kv]


def attention(q, k, v, scale: float, pattern=None, causal: bool = True, q_start: int = 0):
    """Whole-tensor oracle. q [B,n_q,H,dqk], k [B,n_kv,dqk], v [B,n_kv,dv]; pattern (s,l,b) or None (full).
    Returns O [B,n_q,H,dv] fp64 and LSE [B,H,n_q] fp64."""
    B, n_q, H, dqk = q.shape
    dv = v.shape[-1]
    o = np.empty((B, n_q, H, dv), dtype=np.float64)
    lse = np.empty((B, H, n_q), dtype=np.float64)
    s, l, b = pattern if pattern is not None else (0, 1, 1)
    pos = np.repeat(np.arange(q_start, q_start + n_q, dtype=np.int64), H)
    for bi in range(B):
        ob, lb = attention_rows(q[bi].reshape(n_q * H, dqk), pos, k[bi], v[bi], scale, s, l, b,
                                sparse=pattern is not None, causal=causal)
        o[bi] = ob.reshape(n_q, H, dv)
        lse[bi] = lb.reshape(n_q, H).T
    return o, lse


def blend(o, op, alpha: float, dohat=None):
    """Eq. 3: returns (ohat fp64, dalpha fp64 or None)."""
    o, op = _c32(o).ravel(), _c32(op).ravel()
    n = o.size
    ohat = np.empty(n, dtype=np.float64)
    dal = np.zeros(1, dtype=np.float64)
    if dohat is not None:
        dohat = _c32(dohat).ravel()
        lib().loza_oracle_blend(o, op, float(alpha), dohat.ctypes.data, n, ohat.ctypes.data, dal.ctypes.data)
        return ohat, float(dal[0])
    lib().loza_oracle_blend(o, op, float(alpha), None, n, ohat.ctypes.data, None)
    return ohat, None
