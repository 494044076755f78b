"""GPU parity of the tcgen05 bf16 prefill (SSA and full) on the absorbed MLA shape, vs the fp64 oracle.

Tolerance (north star / DESIGN.md §3): bf16 inputs, fp32 accumulation -> max-abs <= 2e-2 on unit-scale data
(binding), plus a normwise guard ||d||_inf / ||O_ref||_inf <= 1e-2 (P is rounded to bf16 before PV).
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_K, TID_Q, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu

D_QK, D_V = 576, 512
SCALE = loza.default_scale(576)
MAXABS = 2e-2
NORMWISE = 1e-2


def _specs(seed, B, n, H, kind="plain", b=128):
    qk = "q_sink" if kind == "sink" else "plain"
    kk = {"sink": "kv_sink", "marker": "kv_marker"}.get(kind, "plain")
    qs = Spec(seed=seed, tensor_id=TID_Q, batch=B, n=n, heads=H, d=D_QK, kind=qk, amp=5.27, col=D_QK - 1)
    ks = Spec(seed=seed, tensor_id=TID_K, batch=B, n=n, heads=1, d=D_QK, kind=kk, amp=5.27 if kind == "sink" else 0.5,
              col=D_QK - 1, sink_rows=b, block=b, marker_mod=D_V)
    return qs, ks


def _check_rows(o, lse, qs, ks, toks, pattern, sparse, bi=0, q_start=0, n_kv=None, causal=True):
    H = qs.heads
    n_kv = n_kv or ks.n
    kf = gen_rows_f32(ks, bi * ks.n, n_kv)
    s, l, b = pattern if sparse else (0, 1, 1)
    worst = 0.0
    for t in toks:
        qr = gen_rows_f32(qs, (bi * qs.n + t) * H, H)
        ref, rl = oracle.attention_rows(qr, np.full(H, q_start + t), kf, kf[:, :D_V], SCALE, s, l, b, sparse=sparse,
                                        causal=causal)
        got = o[bi, t].double().cpu().numpy()
        err = np.abs(got - ref).max()
        worst = max(worst, err)
        assert err <= MAXABS, (t, err)
        assert err / np.abs(ref).max() <= NORMWISE, (t, err)
        if lse is not None:
            gl = lse[bi, :, t].double().cpu().numpy()
            assert np.abs(gl - rl).max() <= 1e-3 * max(1.0, np.abs(rl).max()), t
    return worst


@pytest.mark.parametrize("kind", ["plain", "marker", "sink"])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_ssa_prefill_small(kind, out_dtype):
    n, H, pat = 1024, 64, (1, 2, 128)
    qs, ks = _specs(1, 1, n, H, kind)
    q, kv = empty_filled(qs), empty_filled(ks)
    lse = torch.full((1, H, n), float("nan"), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE, lse=lse, out_dtype=out_dtype)
    torch.cuda.synchronize()
    assert torch.isfinite(o).all()
    _check_rows(o, lse, qs, ks, [0, 1, 63, 127, 128, 255, 256, 300, 383, 384, 511, 640, 1000, 1022, 1023], pat, True)


def test_ssa_prefill_no_sink_blocks():
    """s = 0 (local window only, PAPER.md's SSA with no sink): the tcgen05 prefill against the oracle, LSE too."""
    n, H, pat = 1024, 64, (0, 3, 128)
    qs, ks = _specs(3, 1, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    lse = torch.full((1, H, n), float("nan"), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE, lse=lse, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.isfinite(o).all()
    _check_rows(o, lse, qs, ks, [0, 127, 128, 383, 384, 385, 511, 700, 1023], pat, True)


def test_ssa_paper_pattern_and_window_degeneracy():
    """(1,7,128) at n=2048 vs oracle; and n <= (s+l)b => SSA == full attention (north star)."""
    n, H = 2048, 64
    qs, ks = _specs(2, 1, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    o = loza.ssa_prefill(q, kv, pattern=(1, 7, 128), scale=SCALE, out_dtype=torch.float32)
    torch.cuda.synchronize()
    _check_rows(o, None, qs, ks, [0, 511, 895, 896, 1023, 1024, 1151, 1152, 1500, 2047], (1, 7, 128), True)
    # window covers the whole prefix of the first 1024 tokens: rows < 1024 equal full attention
    of = loza.full_attn_ref(q[:, :1024], kv[:, :1024], scale=SCALE, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.equal(o[:, :1024], of)


def test_full_prefill_causal_and_bidirectional():
    n, H = 1024, 64
    qs, ks = _specs(3, 1, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    lse = torch.empty((1, H, n), device="cuda")
    o = loza.full_attn_ref(q, kv, scale=SCALE, lse=lse, out_dtype=torch.float32)
    ob = loza.full_attn_ref(q, kv, scale=SCALE, causal=False, out_dtype=torch.float32)
    torch.cuda.synchronize()
    _check_rows(o, lse, qs, ks, [0, 1, 127, 128, 700, 1023], None, False)
    _check_rows(ob, None, qs, ks, [0, 500, 1023], None, False, causal=False)


def test_ragged_batched_q_start():
    """batch 2, ragged n (not a multiple of 128), q_start > 0 (queries [q_start, n) against keys [0, n))."""
    B, n, H, pat = 2, 1000, 64, (1, 3, 128)
    qs, ks = _specs(4, B, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    q_start = 384
    o = loza.ssa_prefill(q[:, q_start:], kv, pattern=pat, scale=SCALE, q_start=q_start, out_dtype=torch.float32)
    torch.cuda.synchronize()
    for bi in range(B):
        toks = [0, 1, 127, 128, 400, 614, 615]
        for t in toks:
            qr = gen_rows_f32(qs, (bi * n + q_start + t) * H, H)
            kf = gen_rows_f32(ks, bi * n, n)
            ref, _ = oracle.attention_rows(qr, np.full(H, q_start + t), kf, kf[:, :D_V], SCALE, *pat)
            assert np.abs(o[bi, t].double().cpu().numpy() - ref).max() <= MAXABS


def test_block_size_256():
    n, H, pat = 1536, 64, (1, 2, 256)
    qs, ks = _specs(5, 1, n, H, "marker", b=256)
    q, kv = empty_filled(qs), empty_filled(ks)
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE, out_dtype=torch.float32)
    torch.cuda.synchronize()
    _check_rows(o, None, qs, ks, [0, 127, 128, 255, 256, 383, 384, 511, 512, 767, 768, 1100, 1535], pat, True)


def test_deterministic_and_perturbation_locality():
    """Bitwise-repeatable; perturbing KV rows outside every window of a query block leaves it bitwise unchanged
    (SPEC.md:168)."""
    n, H, pat = 2048, 64, (1, 2, 128)
    qs, ks = _specs(6, 1, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    o1 = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE)
    o2 = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE)
    kv2 = kv.clone()
    kv2[:, 128:1024] += 1.0  # blocks 1..7: outside the window of query blocks >= 9
    o3 = loza.ssa_prefill(q, kv2, pattern=pat, scale=SCALE)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    assert torch.equal(o1[:, 9 * 128:], o3[:, 9 * 128:])
    assert not torch.equal(o1[:, 128:1024], o3[:, 128:1024])


@pytest.mark.slow
def test_ssa_prefill_32k_sampled():
    """BASELINE.json configs[1] at full size (B1 H64 n32768, (1,7,128)), sampled rows, bench launch config."""
    n, H, pat = 32768, 64, (1, 7, 128)
    qs, ks = _specs(0, 1, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    toks = sorted(set([0, 127, 128, 1023, 1024, n - 1] + rng.integers(0, n, 10).tolist()))
    _check_rows(o, None, qs, ks, toks, pat, True)


@pytest.mark.parametrize("world", [2, 4])
def test_seqpar_local_emulation_bf16_mla_bitwise(world):
    """Sequence-parallel prefill (segmented KV [sink | halo | shard] through the tcgen05 kernel) equals the
    single-GPU prefill bitwise; the exchange is emulated with device copies (virtual ranks)."""
    pat = (1, 7, 128)
    n_local = 1024
    n = n_local * world
    qs, ks = _specs(7, 1, n, 64)
    q, kv = empty_filled(qs), empty_filled(ks)
    ref = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE)
    shards = [kv[:, r * n_local:(r + 1) * n_local].contiguous() for r in range(world)]
    for r in range(world):
        o = loza.ssa_seqpar_prefill_local(q[:, r * n_local:(r + 1) * n_local].contiguous(), shards[r], None, pat, SCALE,
                                          rank=r, world=world, rank0_k=shards[0],
                                          prev_k=shards[r - 1] if r > 0 else None)
        torch.cuda.synchronize()
        assert torch.equal(o, ref[:, r * n_local:(r + 1) * n_local]), r


def test_chunked_prefill_bitwise():
    """chunked prefill through q_start (queries [a, e) against the KV prefix [0, e)) equals the whole-sequence
    prefill bit for bit (work units are independent); this is how bench.py's e2e leg pipelines PCIe."""
    n, H, pat, nc = 4096, 64, (1, 7, 128), 1024
    qs, ks = _specs(8, 1, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    ref = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE)
    out = torch.empty_like(ref)
    for a in range(0, n, nc):
        loza.ssa_prefill(q[:, a:a + nc], kv[:, :a + nc], pattern=pat, scale=SCALE, out=out[:, a:a + nc], q_start=a)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("n,H,pat", [(1024, 8, (1, 7, 128)), (256, 128, (1, 1, 128)), (640, 2, (1, 2, 128)),
                                     (200, 16, (1, 7, 128)), (384, 192, (2, 1, 128))])
def test_ssa_prefill_head_counts(n, H, pat):
    """The tcgen05 prefill at other head counts (a 128-row unit then spans 128 / H tokens, or a token spans several
    units): H = 2, 8, 16 (n_q * H % 128 == 0), 128 and 192 (H % 64 == 0); every token against the oracle."""
    qs, ks = _specs(21 + H, 1, n, H)
    q, kv = empty_filled(qs), empty_filled(ks)
    lse = torch.empty((1, H, n), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE, lse=lse, out_dtype=torch.float32)
    torch.cuda.synchronize()
    _check_rows(o, lse, qs, ks, range(n), pat, True)
