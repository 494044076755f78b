"""GPU parity of the tcgen05 split-KV decode (SSA and full) on the absorbed MLA shape, vs the fp64 oracle.

The oracle materialises the mask row at p = seq_len - 1 (DESIGN R8) and attends the allowed rows only; the
rows are regenerated on the host from the counter-based generator (no copy back from the device).
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_K, TID_Q, Spec, gen_rows_f32, gen_rows_f32_at
from inputs.device import empty_filled, fill_
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu

D_QK, D_V, H = 576, 512, 64
SCALE = loza.default_scale(576)
MAXABS = 2e-2


def _oracle_decode(qs, ks, bi, L, pattern, sparse=True):
    s, l, b = pattern if sparse else (0, 1, 1)
    keys = oracle.allowed_keys(L - 1, L, s, l, b, sparse=sparse)
    kf = gen_rows_f32_at(ks, bi * ks.n + keys)
    qr = gen_rows_f32(qs, bi * H, H)
    return oracle.attend(qr, kf, kf[:, :D_V], SCALE)


@pytest.mark.parametrize("pattern", [(1, 7, 128), (1, 2, 128), (2, 3, 256), (0, 3, 128)])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_ssa_decode_ragged(pattern, out_dtype):
    seq = [1, 100, 128, 129, 1023, 1024, 1025, 2048, 3000, 4096]
    B, T = len(seq), 4096
    qs = Spec(seed=3, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    ks = Spec(seed=3, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK, kind="kv_marker", block=pattern[2],
              marker_mod=D_V, amp=0.5)
    q, cache = empty_filled(qs), empty_filled(ks)
    sl = torch.tensor(seq, dtype=torch.int32, device="cuda")
    lse = torch.full((B, H, 1), float("nan"), device="cuda")
    o = loza.ssa_decode(q, cache, sl, pattern=pattern, scale=SCALE, out_dtype=out_dtype, lse=lse)
    torch.cuda.synchronize()
    for bi, L in enumerate(seq):
        ref, rl = _oracle_decode(qs, ks, bi, L, pattern)
        got = o[bi, 0].double().cpu().numpy()
        assert np.abs(got - ref).max() <= MAXABS, (bi, L, np.abs(got - ref).max())
        assert np.abs(lse[bi, :, 0].double().cpu().numpy() - rl).max() <= 1e-3 * max(1, np.abs(rl).max())


def test_full_decode_ragged():
    seq = [1, 130, 777, 4096, 5000, 9000]
    B, T = len(seq), 9000
    qs = Spec(seed=4, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    ks = Spec(seed=4, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    q, cache = empty_filled(qs), empty_filled(ks)
    sl = torch.tensor(seq, dtype=torch.int32, device="cuda")
    o = loza.full_attn_ref(q, cache, scale=SCALE, seq_lens=sl, out_dtype=torch.float32)
    torch.cuda.synchronize()
    for bi, L in enumerate(seq):
        ref, _ = _oracle_decode(qs, ks, bi, L, None, sparse=False)
        assert np.abs(o[bi, 0].double().cpu().numpy() - ref).max() <= MAXABS, (bi, L)


def test_decode_equals_last_prefill_row():
    """Streaming equivalence: decode at seq_len t == row t-1 of the prefill over t tokens."""
    n = 2048
    qs = Spec(seed=5, tensor_id=TID_Q, batch=1, n=n, heads=H, d=D_QK)
    ks = Spec(seed=5, tensor_id=TID_K, batch=1, n=n, heads=1, d=D_QK)
    q, kv = empty_filled(qs), empty_filled(ks)
    op = loza.ssa_prefill(q, kv, pattern=(1, 7, 128), scale=SCALE, out_dtype=torch.float32)
    for t in (1, 128, 129, 1024, 1500, 2048):
        od = loza.ssa_decode(q[:, t - 1:t].contiguous(), kv, torch.tensor([t], dtype=torch.int32, device="cuda"),
                             pattern=(1, 7, 128), scale=SCALE, out_dtype=torch.float32)
        torch.cuda.synchronize()
        assert float((od[0, 0] - op[0, t - 1]).abs().max()) <= 1e-2, t


def test_context_independence_bitwise():
    """Equal sink + window contents at 128K and at 1M context give bit-identical SSA decode outputs."""
    B, T = 2, 1 << 20
    ks = Spec(seed=6, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    qs = Spec(seed=6, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    cache = torch.empty((B, T, D_QK), dtype=torch.bfloat16, device="cuda")
    fill_(cache, ks)
    q = empty_filled(qs)
    w = 7 * 128
    t1, t2 = 131072, T
    cache[:, t2 - w:t2] = cache[:, t1 - w:t1]
    o1 = loza.ssa_decode(q, cache, torch.full((B,), t1, dtype=torch.int32, device="cuda"), scale=SCALE)
    o2 = loza.ssa_decode(q, cache, torch.full((B,), t2, dtype=torch.int32, device="cuda"), scale=SCALE)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)


@pytest.mark.slow
def test_ssa_decode_bench_config_sampled():
    """BASELINE.json configs[3]: B64 H64, context 128K, in the bench launch configuration; sampled sequences."""
    B, T = 64, 131072
    ks = Spec(seed=0, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    qs = Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    cache = torch.empty((B, T, D_QK), dtype=torch.bfloat16, device="cuda")
    fill_(cache, ks)
    q = empty_filled(qs)
    sl = torch.full((B,), T, dtype=torch.int32, device="cuda")
    sl[5] = T - 77  # ragged
    o = loza.ssa_decode(q, cache, sl, scale=SCALE)
    of = loza.full_attn_ref(q, cache, scale=SCALE, seq_lens=sl)
    torch.cuda.synchronize()
    for bi in (0, 5, 31, 63):
        L = int(sl[bi])
        ref, _ = _oracle_decode(qs, ks, bi, L, (1, 7, 128))
        assert np.abs(o[bi, 0].double().cpu().numpy() - ref).max() <= MAXABS, bi
    for bi in (0, 63):
        ref, _ = _oracle_decode(qs, ks, bi, int(sl[bi]), None, sparse=False)
        assert np.abs(of[bi, 0].double().cpu().numpy() - ref).max() <= MAXABS, bi


@pytest.mark.parametrize("B", [74, 80])
def test_ssa_decode_large_batch(B):
    """B = 74 is the largest batch on the pair kernels (2 CTAs per sequence on 148 SMs); B = 80 runs the
    flattened split-KV kernel. Ragged seq_lens, sampled sequences against the oracle."""
    T = 2048
    pattern = (1, 7, 128)
    rng = np.random.default_rng(80 + B)
    seq = [int(x) for x in rng.integers(1, T + 1, B)]
    seq[0], seq[-1] = 1, T
    qs = Spec(seed=12, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    ks = Spec(seed=12, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    q, cache = empty_filled(qs), empty_filled(ks)
    sl = torch.tensor(seq, dtype=torch.int32, device="cuda")
    o = loza.ssa_decode(q, cache, sl, pattern=pattern, scale=SCALE)
    torch.cuda.synchronize()
    for bi in sorted({0, B - 1, *[int(x) for x in rng.integers(0, B, 6)]}):
        ref, _ = _oracle_decode(qs, ks, bi, seq[bi], pattern)
        got = o[bi, 0].double().cpu().numpy()
        assert np.abs(got - ref).max() <= MAXABS, (bi, seq[bi], np.abs(got - ref).max())


@pytest.mark.parametrize("pattern,heads", [((1, 7, 128), 64), ((2, 3, 256), 64), ((1, 7, 128), 32)])
def test_ssa_decode_rescale_in_later_tiles(pattern, heads):
    """The running per-head max grows past the lazy-rescale threshold (2^8) twice after the first tile: the
    RoPE column of every query and of the keys of two later selected blocks is raised (host-side input
    construction from the numpy generator twin), so O^T and the row sums are rescaled in tiles >= 2 while S runs
    ahead of PV (H = 64: the pair-cooperative kernel; H = 32: the key-split kernel of a head-sharded GPU).
    Eq. 4 against the fp64 oracle on exactly the uploaded bf16 values."""
    s, l, b = pattern
    B, T, Hh = 3, 4096, heads
    qs = Spec(seed=21, tensor_id=TID_Q, batch=B, n=1, heads=Hh, d=D_QK)
    ks = Spec(seed=21, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    qf = gen_rows_f32(qs, 0, B * Hh).reshape(B, Hh, D_QK)
    kf = gen_rows_f32(ks, 0, B * T).reshape(B, T, D_QK)
    seq = [T, T - 100, 3000]
    qf[:, :, D_QK - 1] += 12.0
    for bi, L in enumerate(seq):
        qb = (L - 1) // b
        lo = max(s, qb - l + 1)  # first local block
        mid = lo + (qb - lo) // 2
        kf[bi, mid * b:(mid + 1) * b, D_QK - 1] += 12.0  # a later tile: the max jumps by ~144 scale log2(e) ~ 15
        kf[bi, qb * b:L, D_QK - 1] += 20.0               # the last block: jumps again (~25)
    q = torch.from_numpy(qf).to(torch.bfloat16).reshape(B, 1, Hh, D_QK).cuda()
    cache = torch.from_numpy(kf).to(torch.bfloat16).cuda()
    qh = q.float().cpu().numpy().astype(np.float64).reshape(B, Hh, D_QK)
    kh = cache.float().cpu().numpy().astype(np.float64)
    sl = torch.tensor(seq, dtype=torch.int32, device="cuda")
    lse = torch.full((B, Hh, 1), float("nan"), device="cuda")
    o = loza.ssa_decode(q, cache, sl, pattern=pattern, scale=SCALE, out_dtype=torch.float32, lse=lse)
    torch.cuda.synchronize()
    for bi, L in enumerate(seq):
        keys = oracle.allowed_keys(L - 1, L, s, l, b)
        ref, rl = oracle.attend(qh[bi], kh[bi, keys], kh[bi, keys][:, :D_V], SCALE)
        got = o[bi, 0].double().cpu().numpy()
        assert np.abs(got - ref).max() <= MAXABS, (bi, L, np.abs(got - ref).max())
        assert np.abs(lse[bi, :, 0].double().cpu().numpy() - rl).max() <= 1e-3 * max(1, np.abs(rl).max())
