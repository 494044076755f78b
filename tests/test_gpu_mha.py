"""GPU parity of ssa_prefill_mha, the non-absorbed (MHA-form) SSA prefill: per head h,
O_h = Eq. 4 over (q_h, k_h, v_h) with d_qk 192 (128 nope + 64 RoPE) and d_v 128 - compared, head by head,
with oracle.attention_rows (fp64, pinned in tests/test_oracle_pins.py) on the same bf16-rounded inputs.

Tolerance (R12): bf16 output <= 2e-2 max-abs (P is rounded to bf16 before PV, O to bf16 at the
end); fp32 output and LSE <= 1e-2 (P rounding only).
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_K, TID_Q, TID_V, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu

DQK, DV = 192, 128


def _inputs(seed, B, n, H, n_kv=None):
    n_kv = n if n_kv is None else n_kv
    qs = Spec(seed=seed, tensor_id=TID_Q, batch=B, n=n, heads=H, d=DQK)
    ks = Spec(seed=seed, tensor_id=TID_K, batch=B, n=n_kv, heads=H, d=DQK)
    vs = Spec(seed=seed, tensor_id=TID_V, batch=B, n=n_kv, heads=H, d=DV)
    return (qs, ks, vs), tuple(empty_filled(s, four_d=True) for s in (qs, ks, vs))


def _ref_head(specs, bi, h, rows, pat, scale, q_start=0, sparse=True, causal=True):
    """oracle rows of head h, batch bi, for local query rows `rows`"""
    qs, ks, vs = specs
    H, n, n_kv = qs.heads, qs.n, ks.n
    qa = gen_rows_f32(qs, bi * n * H, n * H).reshape(n, H, DQK)[rows, h]
    ka = gen_rows_f32(ks, bi * n_kv * H, n_kv * H).reshape(n_kv, H, DQK)[:, h]
    va = gen_rows_f32(vs, bi * n_kv * H, n_kv * H).reshape(n_kv, H, DV)[:, h]
    return oracle.attention_rows(qa, q_start + np.asarray(rows), ka, va, scale, *pat, sparse=sparse, causal=causal)


@pytest.mark.parametrize("B,n,H,pat", [(2, 1000, 4, (1, 2, 128)), (1, 1536, 2, (2, 1, 256)), (1, 129, 3, (1, 7, 128)),
                                      (1, 900, 2, (0, 2, 128)), (1, 1200, 2, (1, 2, 384))])
def test_mha_ssa_all_rows(B, n, H, pat):
    specs, (q, k, v) = _inputs(61, B, n, H)
    scale = 1.0 / np.sqrt(DQK)
    lse = torch.empty((B, H, n), device="cuda")
    o = loza.ssa_prefill_mha(q, k, v, pat, scale, lse=lse)
    torch.cuda.synchronize()
    for bi in range(B):
        for h in range(H):
            ref, rl = _ref_head(specs, bi, h, np.arange(n), pat, scale)
            got = o[bi, :, h].double().cpu().numpy()
            assert np.abs(got - ref).max() <= 2e-2, (bi, h)
            assert np.abs(lse[bi, h].double().cpu().numpy() - rl).max() <= 1e-2, (bi, h)


@pytest.mark.parametrize("causal", [True, False])
def test_mha_full_comparator(causal):
    B, n, H = 1, 700, 2
    specs, (q, k, v) = _inputs(62, B, n, H)
    scale = 0.07
    o = loza.ssa_prefill_mha(q, k, v, scale=scale, sparse=False, causal=causal, out_dtype=torch.float32)
    torch.cuda.synchronize()
    for h in range(H):
        ref, _ = _ref_head(specs, 0, h, np.arange(n), (0, 1, 1), scale, sparse=False, causal=causal)
        assert np.abs(o[0, :, h].double().cpu().numpy() - ref).max() <= 1e-2, h


def test_mha_strided_layouts():
    """k | v fused per head ([B, n, H, 320], the up-projection's output), q as a [B, H, n, d] buffer viewed as
    [B, n, H, d]; o written into a [B, H, n, 128] buffer's permuted view. Equal bitwise to the packed call."""
    B, n, H = 2, 640, 4
    pat = (1, 2, 128)
    specs, (q, k, v) = _inputs(63, B, n, H)
    ref = loza.ssa_prefill_mha(q, k, v, pat)
    kv = torch.cat([k, v], dim=-1)
    qt = q.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
    ot = torch.empty((B, H, n, DV), dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
    loza.ssa_prefill_mha(qt, kv[..., :DQK], kv[..., DQK:], pat, out=ot)
    torch.cuda.synchronize()
    assert torch.equal(ot, ref)


def test_mha_chunked_prefill_bitwise():
    """queries in chunks [q0, q0 + c) against keys [0, q0 + c) equal the whole prefill bitwise."""
    B, n, H = 1, 2048, 2
    pat = (1, 3, 128)
    _, (q, k, v) = _inputs(64, B, n, H)
    ref = loza.ssa_prefill_mha(q, k, v, pat)
    for q0, c in [(0, 384), (384, 640), (1024, 1024)]:
        o = loza.ssa_prefill_mha(q[:, q0:q0 + c], k[:, :q0 + c], v[:, :q0 + c], pat, q_start=q0)
        torch.cuda.synchronize()
        assert torch.equal(o, ref[:, q0:q0 + c]), q0


def test_mha_paper_pattern_sampled():
    """(1,7,128) over 4096 tokens, H = 8: sampled rows per head (first block, block edges, the tail)."""
    B, n, H = 1, 4096, 8
    pat = (1, 7, 128)
    specs, (q, k, v) = _inputs(65, B, n, H)
    scale = 1.0 / np.sqrt(DQK)
    o = loza.ssa_prefill_mha(q, k, v, pat, scale)
    torch.cuda.synchronize()
    rows = np.array([0, 127, 128, 1023, 1024, 1151, 2047, 3000, 4095])
    for h in range(H):
        ref, _ = _ref_head(specs, 0, h, rows, pat, scale)
        assert np.abs(o[0, rows, h].double().cpu().numpy() - ref).max() <= 2e-2, h


def test_mha_degenerate_and_errors():
    _, (q, k, v) = _inputs(66, 1, 256, 2)
    o = loza.ssa_prefill_mha(q[:, :0], k, v)  # n_q == 0
    assert o.shape == (1, 0, 2, DV)
    o1 = loza.ssa_prefill_mha(q[:, :1], k[:, :1], v[:, :1], out_dtype=torch.float32)  # one token: O ~= v_0
    torch.cuda.synchronize()
    assert torch.allclose(o1[0, 0], v[0, 0].float(), atol=1e-2, rtol=0)
    with pytest.raises(loza.LozaError, match="UNSUPPORTED"):
        loza.ssa_prefill_mha(q, k, v, (1, 2, 64))  # b % 128 != 0
    with pytest.raises(loza.LozaError, match="UNSUPPORTED"):
        loza.ssa_prefill_mha(q[..., :128].contiguous(), k[..., :128].contiguous(), v)  # d_qk != 192
    with pytest.raises(loza.LozaError, match="SHAPE"):
        loza.ssa_prefill_mha(q, k[:, :100], v[:, :100])  # n_kv < q_start + n_q
