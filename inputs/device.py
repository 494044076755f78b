"""Device-side fill through inputs/libloza_gen.so (the CUDA twin of gen.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess

from .gen import Spec, stream_key  # noqa: F401  (re-exported for callers)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libloza_gen.so")
SRC = os.path.join(_HERE, "csrc", "loza_gen.cu")


class _GenSpec(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("tensor_id", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("batch", ctypes.c_int64), ("n", ctypes.c_int64), ("heads", ctypes.c_int64),
                ("d", ctypes.c_int64), ("kind", ctypes.c_int32), ("block", ctypes.c_int32),
                ("marker_mod", ctypes.c_int32), ("col", ctypes.c_int32), ("sink_rows", ctypes.c_int64),
                ("amp", ctypes.c_float)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC):
        cmd = ["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
               "-lineinfo", SRC, "-o", LIB_PATH]
        subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        lib.loza_gen_fill.restype = ctypes.c_int
        lib.loza_gen_fill.argtypes = [ctypes.c_void_p, ctypes.POINTER(_GenSpec), ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_void_p]
        _lib = lib
    return _lib


def _cspec(spec: Spec) -> _GenSpec:
    return _GenSpec(spec.seed, spec.tensor_id, 1 if spec.dtype == "bf16" else 0, spec.batch, spec.n,
                    spec.heads, spec.d, spec.kind_id(), spec.block, spec.marker_mod, spec.col,
                    spec.sink_rows, spec.amp)


def fill_(t, spec: Spec, row_start: int = 0) -> None:
    """Write rows [row_start, row_start + t.numel()/d) of ``spec`` into contiguous CUDA tensor t."""
    import torch
    assert t.is_cuda and t.is_contiguous()
    assert t.dtype == (torch.bfloat16 if spec.dtype == "bf16" else torch.float32)
    assert t.numel() % spec.d == 0
    rows = t.numel() // spec.d
    cs = _cspec(spec)
    stream = torch.cuda.current_stream(t.device).cuda_stream
    rc = _load().loza_gen_fill(ctypes.c_void_p(t.data_ptr()), ctypes.byref(cs), row_start, rows,
                               ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"loza_gen_fill failed with code {rc}")


def empty_filled(spec: Spec, device="cuda", four_d: bool | None = None):
    """Allocate the tensor on the device and fill it from the generator: [batch, n, heads, d] for query-like
    tensors (heads > 1 or tensor_id == TID_Q), else [batch, n, d]."""
    import torch
    from .gen import TID_Q
    dt = torch.bfloat16 if spec.dtype == "bf16" else torch.float32
    if four_d is None:
        four_d = spec.heads > 1 or spec.tensor_id == TID_Q
    shape = (spec.batch, spec.n, spec.heads, spec.d) if four_d else (spec.batch, spec.n, spec.d)
    t = torch.empty(shape, dtype=dt, device=device)
    fill_(t, spec)
    return t
