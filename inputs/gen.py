"""Seeded, counter-based synthetic input generator (host side, numpy).

This module is shared by the CPU oracle side and the CUDA side of the test
suite and the bench. It holds NONE of the method's arithmetic (no masks, no
softmax, no attention): it only turns (seed, tensor id, flat element index)
into a value, so any element of a tensor of any size can be regenerated
without materialising the tensor (e.g. one KV row out of a 1.2 GB cache).

The CUDA twin lives in ``inputs/csrc/loza_gen.cu`` and implements the same
integer / IEEE-fp32 recipe, element by element; ``tests/test_gen_gpu.py``
checks the two bitwise.

Recipe (DESIGN.md §"Input recipe"):
  key   = mix(seed * G ^ (tensor_id * C))
  bits  = mix(key + (index + 1) * G)                  (splitmix64 finaliser)
  s     = sum of the four 16-bit fields of bits        (Irwin-Hall, n=4)
  z     = fp32(s - 131070) * fp32(sqrt(3)/65536)       (one IEEE RN multiply)
          -> mean 0, variance 1 (up to 2^-32), support |z| <= 3.46
  z    += structure term (fp32 RN add), see ``Spec.kind``
  value = z (fp32) or bf16_rne(z)

Structures (SURVEY.md §8 d, "Value distributions"):
  plain       D1: iid ~N(0,1)-like, unit scale (the north-star tolerance data)
  kv_marker   D3: KV row at position j gets +amp on coordinate (j // b) % d_v
              (a wrong or missing key block shifts a known output coordinate)
  kv_sink     D2: KV rows of the first ``sink_rows`` positions get +amp on
              coordinate ``col`` (an attention-sink direction)
  q_sink      D2: every query row gets +amp on coordinate ``col``
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
TID_MUL = 0xD1B54A32D192ED03
NORM_SCALE_BITS = 0x37DDB3D7  # fp32(sqrt(3)/65536)
NORM_SCALE = np.array([NORM_SCALE_BITS], dtype=np.uint32).view(np.float32)[0]

# tensor ids (shared with loza_gen.cu)
TID_Q = 1
TID_K = 2      # K, or the latent KV cache for MLA (V aliases its first d_v columns)
TID_V = 3      # separate V (non-MLA shapes only)
TID_DO = 4     # upstream gradient dO_hat for the blend
TID_O_FULL = 5
TID_O_SPARSE = 6

KIND_PLAIN = 0
KIND_KV_MARKER = 1
KIND_KV_SINK = 2
KIND_Q_SINK = 3
_KINDS = {"plain": KIND_PLAIN, "kv_marker": KIND_KV_MARKER,
          "kv_sink": KIND_KV_SINK, "q_sink": KIND_Q_SINK}


def _mix_scalar(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def stream_key(seed: int, tensor_id: int) -> int:
    return _mix_scalar(((seed * GOLDEN) ^ (tensor_id * TID_MUL)) & MASK64)


@dataclass(frozen=True)
class Spec:
    """Logical tensor [batch, n, heads, d] (heads=1 for K/KV/V rows)."""
    seed: int
    tensor_id: int
    batch: int
    n: int
    heads: int
    d: int
    dtype: str = "bf16"          # "bf16" | "f32"
    kind: str = "plain"
    block: int = 128             # b, for kv_marker
    marker_mod: int = 512        # d_v, for kv_marker
    amp: float = 0.0
    col: int = 0                 # coordinate for kv_sink / q_sink
    sink_rows: int = 0           # rows (positions) boosted by kv_sink

    @property
    def numel(self) -> int:
        return self.batch * self.n * self.heads * self.d

    @property
    def rows(self) -> int:
        return self.batch * self.n * self.heads

    def kind_id(self) -> int:
        return _KINDS[self.kind]


def raw_normal(seed: int, tensor_id: int, idx: np.ndarray) -> np.ndarray:
    """fp32 unit-variance value for each flat index (no structure, no rounding to bf16)."""
    key = np.uint64(stream_key(seed, tensor_id))
    with np.errstate(over="ignore"):
        x = key + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
    bits = _mix(x)
    s = (bits & np.uint64(0xFFFF)) + ((bits >> np.uint64(16)) & np.uint64(0xFFFF)) \
        + ((bits >> np.uint64(32)) & np.uint64(0xFFFF)) + (bits >> np.uint64(48))
    zi = s.astype(np.int64) - 131070
    return zi.astype(np.float32) * NORM_SCALE  # exact int->fp32, one RN multiply


def bf16_rne_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return u.astype(np.uint16)


def bf16_bits_to_f32(u: np.ndarray) -> np.ndarray:
    return (u.astype(np.uint32) << np.uint32(16)).view(np.float32)


def gen_rows_f32(spec: Spec, row_start: int, row_count: int) -> np.ndarray:
    """Rows [row_start, row_start+row_count) of the flat [batch*n*heads, d] view,
    as fp32 values exactly equal to what the device holds (bf16 widened exactly)."""
    return gen_rows_f32_at(spec, np.arange(row_start, row_start + row_count, dtype=np.int64))


def gen_rows_f32_at(spec: Spec, rows) -> np.ndarray:
    """Arbitrary rows (flat [batch*n*heads] indices) as fp32 values, shape [len(rows), d]."""
    d = spec.d
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    row_count = len(rows)
    cols = np.arange(d, dtype=np.int64)
    idx = rows[:, None] * d + cols[None, :]
    z = raw_normal(spec.seed, spec.tensor_id, idx)
    kind = spec.kind_id()
    if kind != KIND_PLAIN:
        pos = (rows // spec.heads) % spec.n
        amp = np.float32(spec.amp)
        if kind == KIND_KV_MARKER:
            hit = cols[None, :] == ((pos // spec.block) % spec.marker_mod)[:, None]
        elif kind == KIND_KV_SINK:
            hit = (cols[None, :] == spec.col) & (pos < spec.sink_rows)[:, None]
        else:  # KIND_Q_SINK
            hit = np.broadcast_to(cols[None, :] == spec.col, z.shape)
        z = np.where(hit, z + amp, z).astype(np.float32)  # fp32 RN add
    if spec.dtype == "bf16":
        return bf16_bits_to_f32(bf16_rne_bits(z)).reshape(row_count, d)
    return z.reshape(row_count, d)


def gen_rows_bits(spec: Spec, row_start: int, row_count: int) -> np.ndarray:
    """Same rows as storage bits: uint16 for bf16, float32 for f32."""
    v = gen_rows_f32(spec, row_start, row_count)
    if spec.dtype == "bf16":
        return bf16_rne_bits(v)
    return v


def gen_f32(spec: Spec) -> np.ndarray:
    """Whole tensor as fp32 values, shape [batch, n, heads, d] (small tensors only)."""
    return gen_rows_f32(spec, 0, spec.rows).reshape(spec.batch, spec.n, spec.heads, spec.d)


def gen_torch(spec: Spec, device="cpu"):
    """Whole tensor as a torch tensor of the spec's dtype (built on the host; small tensors)."""
    import torch
    bits = gen_rows_bits(spec, 0, spec.rows).reshape(spec.batch, spec.n, spec.heads, spec.d)
    if spec.dtype == "bf16":
        t = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16)
    else:
        t = torch.from_numpy(bits)
    return t.to(device)
