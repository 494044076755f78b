"""Degenerate and boundary inputs through every C-ABI entry point (§8(b)): empty batches / sequences are no-ops
that return LOZA_OK and leave outputs untouched, one-token problems reduce to closed forms (softmax over one
key: O = v_0, zero gradients through the softmax for dq / dk of a single key), and the smallest ragged shapes
agree with the oracle."""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_DO, TID_K, TID_Q, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu
H, DQK, DV = 64, 576, 512


def _qkv(n, B=1, seed=90):
    qs = Spec(seed=seed, tensor_id=TID_Q, batch=B, n=n, heads=H, d=DQK)
    ks = Spec(seed=seed, tensor_id=TID_K, batch=B, n=n, heads=1, d=DQK)
    return qs, ks, empty_filled(qs), empty_filled(ks)


def test_prefill_empty_and_single_token():
    _, _, q, kv = _qkv(256)
    sentinel = torch.full((1, 0, H, DV), 7.0, dtype=torch.bfloat16, device="cuda")
    o = loza.ssa_prefill(q[:, :0], kv, out=sentinel)  # n_q == 0: nothing to do
    assert o.shape == (1, 0, H, DV)
    # one query token at position 0 sees only key 0: O = v_0 for every head (P = exp2(s - m) with m taken in
    # another rounding order: 1 within a few ulp, so O = v_0 to fp32 rounding)
    o1 = loza.ssa_prefill(q[:, :1].contiguous(), kv[:, :1].contiguous(), out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.allclose(o1[0, 0], kv[0, 0, :DV].float().expand(H, DV), rtol=1e-5, atol=0)
    # the comparator agrees on the one-token problem
    of = loza.full_attn_ref(q[:, :1].contiguous(), kv[:, :1].contiguous(), out_dtype=torch.float32)
    assert torch.allclose(of, o1, rtol=1e-5, atol=0)


def test_decode_single_key_and_empty_batch():
    _, _, q, kv = _qkv(256)
    qd = q[:, :1].contiguous()
    seq = torch.ones(1, dtype=torch.int32, device="cuda")  # context of one token: O = v_0
    o = loza.ssa_decode(qd, kv, seq, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert torch.allclose(o[0, 0], kv[0, 0, :DV].float().expand(H, DV), rtol=1e-5, atol=0)
    o0 = loza.ssa_decode(qd[:0], kv[:0], seq[:0])  # batch 0
    assert o0.shape[0] == 0


def test_backward_single_token_and_empty():
    qs, ks, q, kv = _qkv(128)
    dos = Spec(seed=91, tensor_id=TID_DO, batch=1, n=128, heads=H, d=DV)
    do = empty_filled(dos)
    q1, k1, d1 = q[:, :1].contiguous(), kv[:, :1].contiguous(), do[:, :1].contiguous()
    lse = torch.empty((1, H, 1), device="cuda")
    o = loza.ssa_prefill(q1, k1, lse=lse)
    dq, dk, dv = loza.attention_backward(q1, k1, o, lse, d1)
    torch.cuda.synchronize()
    # one key: P = 1, dS = P (dP - D) = dO.v - dO.o = 0 up to o's bf16 rounding; dV = sum over heads of dO
    assert float(dq.abs().max()) < 1e-2 and float(dk.abs().max()) < 1e-2
    ref_dv = d1[0, 0].float().sum(0)
    assert torch.allclose(dv[0, 0], ref_dv, atol=1e-3, rtol=1e-3)
    # n_q == 0: empty gradients, dk / dv of the keys are zeros
    lse0 = torch.empty((1, H, 0), device="cuda")
    o0 = torch.empty((1, 0, H, DV), dtype=torch.bfloat16, device="cuda")
    do0 = torch.empty((1, 0, H, DV), dtype=torch.bfloat16, device="cuda")
    dq0, dk0, dv0 = loza.attention_backward(q[:, :0], kv, o0, lse0, do0)
    torch.cuda.synchronize()
    assert dq0.numel() == 0 and float(dk0.abs().max()) == 0.0 and float(dv0.abs().max()) == 0.0


def test_blend_empty_and_ring_append_nothing():
    z = torch.empty(0, dtype=torch.bfloat16, device="cuda")
    alpha = torch.full((1,), 0.5, device="cuda")
    out, _ = loza.loza_blend(z, z, alpha)
    assert out.numel() == 0
    pat = (1, 7, 128)
    cache = torch.full((1, loza.ring_rows(pat), DQK), 3.0, dtype=torch.bfloat16, device="cuda")
    before = cache.clone()
    loza.ssa_ring_append(cache, torch.empty((1, 0, DQK), dtype=torch.bfloat16, device="cuda"),
                         torch.zeros(1, dtype=torch.int32, device="cuda"), pat)
    torch.cuda.synchronize()
    assert torch.equal(cache, before)


def test_select_blocks_small():
    idx, cnt = loza.ssa_select_blocks(1, 0, (1, 7, 128))  # one token: its own block only
    torch.cuda.synchronize()
    assert cnt.cpu().tolist() == [1] and idx.cpu()[0, 0].item() == 0


def test_ragged_tiny_prefill_vs_oracle():
    """n = 130 tokens (two blocks, the second with 2 rows), H = 64: every row against the oracle."""
    n = 130
    qs, ks, q, kv = _qkv(n, seed=92)
    o = loza.ssa_prefill(q, kv, pattern=(1, 1, 128), out_dtype=torch.float32)
    torch.cuda.synchronize()
    kf = gen_rows_f32(ks, 0, n)
    ref, _ = oracle.attention_rows(gen_rows_f32(qs, 0, n * H), np.repeat(np.arange(n), H), kf, kf[:, :DV],
                                   loza.default_scale(DQK), 1, 1, 128, sparse=True, causal=True)
    got = o[0].reshape(n * H, DV).double().cpu().numpy()
    assert np.abs(got - ref).max() <= 2e-2


@pytest.mark.parametrize("n,Hh,pat", [(130, 64, (1, 7, 128)), (257, 8, (1, 7, 128)), (200, 1, (1, 2, 128)),
                                      (384, 16, (2, 3, 128)), (129, 64, (0, 3, 128)), (1, 64, (1, 7, 128))])
def test_backward_small_shapes_vs_oracle(n, Hh, pat):
    """Short and ragged SSA backward problems (a partial last block, one head, no sink blocks, two sink blocks,
    a single token) through the default path (CTA-pair key kernels with row splits, dQ GEMM): every dQ row and
    every dK / dV row against the fp64 oracle backward (2e-2 normwise)."""
    qs = Spec(seed=93, tensor_id=TID_Q, batch=1, n=n, heads=Hh, d=DQK)
    ks = Spec(seed=93, tensor_id=TID_K, batch=1, n=n, heads=1, d=DQK)
    dos = Spec(seed=93, tensor_id=TID_DO, batch=1, n=n, heads=Hh, d=DV)
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(dos)
    scale = loza.default_scale(DQK)
    kf = gen_rows_f32(ks, 0, n)
    # O and LSE from the oracle forward (the bf16 prefill takes n_q * H % 128 == 0 or H % 64 == 0 only)
    orow, lrow = oracle.attention_rows(gen_rows_f32(qs, 0, n * Hh), np.repeat(np.arange(n), Hh), kf, kf[:, :DV],
                                       scale, *pat, sparse=True, causal=True)
    o = torch.from_numpy(orow.reshape(1, n, Hh, DV)).to(torch.bfloat16).cuda()
    lse = torch.from_numpy(lrow.reshape(n, Hh).T.copy()[None]).float().cuda()
    dq, dk, dv = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
    torch.cuda.synchronize()
    rq, rk, rv = oracle.attention_backward(gen_rows_f32(qs, 0, n * Hh), np.repeat(np.arange(n), Hh), kf, kf[:, :DV],
                                           gen_rows_f32(dos, 0, n * Hh), scale, *pat, sparse=True, causal=True)

    # normwise, floored at 1e-3 of the dV norm: with one key (n = 1) dq and dk are exactly 0 in the oracle and
    # bf16 rounding of o leaves ~1e-8 (dS = P (dO.v - dO.o))
    floor = 1e-3 * np.linalg.norm(rv)

    def err(got, ref):
        return np.linalg.norm(got - ref) / max(np.linalg.norm(ref), floor)

    assert err(dq[0].reshape(-1, DQK).double().cpu().numpy(), rq) <= 2e-2
    assert err(dk[0].double().cpu().numpy(), rk) <= 2e-2
    assert err(dv[0].double().cpu().numpy(), rv) <= 2e-2
