"""GPU parity of the fused calibration forward `ssa_prefill_blend`: Eq. 3
applied in the SSA prefill epilogue with O' = SSA(Q, KV) (Eq. 4) never written to HBM.

Checks: alpha in {0, 1} bitwise (alpha = 0 == ssa_prefill's bf16 output, alpha = 1 == o_full); o_hat against the
fp64 oracle (SSA rows from the explicit mask, Eq. 3 blend in fp64) within the bf16 tolerance; d_alpha against the
oracle's Eq. 3 gradient evaluated on the very fp32 O' the kernel blends (ssa_prefill with fp32 output computes
the identical fp32 values), within 1e-4 * sum |dO_hat (O - O')| (R12); determinism; bad alpha.
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_DO, TID_K, TID_O_FULL, TID_Q, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu

D_QK, D_V, H = 576, 512, 64
SCALE = loza.default_scale(576)
PAT = (1, 2, 128)


def _inputs(seed, n, B=1):
    qs = Spec(seed=seed, tensor_id=TID_Q, batch=B, n=n, heads=H, d=D_QK)
    ks = Spec(seed=seed, tensor_id=TID_K, batch=B, n=n, heads=1, d=D_QK)
    # o_full: any bf16 tensor of o's layout (the blend is defined for every O); d_o_hat likewise
    ofs = Spec(seed=seed, tensor_id=TID_O_FULL, batch=B, n=n, heads=H, d=D_V)
    dhs = Spec(seed=seed, tensor_id=TID_DO, batch=B, n=n, heads=H, d=D_V)
    return qs, ks, ofs, dhs


def _alpha(a):
    return torch.tensor([a], dtype=torch.float32, device="cuda")


@pytest.mark.parametrize("n", [1024, 1000])
def test_alpha_endpoints_bitwise(n):
    qs, ks, ofs, dhs = _inputs(21, n)
    q, kv, of = empty_filled(qs), empty_filled(ks), empty_filled(ofs)
    ref = loza.ssa_prefill(q, kv, pattern=PAT, scale=SCALE)
    o0, _ = loza.ssa_prefill_blend(q, kv, of, _alpha(0.0), pattern=PAT, scale=SCALE)
    o1, _ = loza.ssa_prefill_blend(q, kv, of, _alpha(1.0), pattern=PAT, scale=SCALE)
    torch.cuda.synchronize()
    assert torch.equal(o0, ref)
    assert torch.equal(o1, of)


@pytest.mark.parametrize("alpha", [0.25, 0.7])
def test_o_hat_and_d_alpha_vs_oracle(alpha):
    n = 1024
    qs, ks, ofs, dhs = _inputs(22, n)
    q, kv, of, dh = (empty_filled(s) for s in (qs, ks, ofs, dhs))
    st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    oh, da = loza.ssa_prefill_blend(q, kv, of, _alpha(alpha), dh, pattern=PAT, scale=SCALE, status=st)
    o_sp32 = loza.ssa_prefill(q, kv, pattern=PAT, scale=SCALE, out_dtype=torch.float32)  # the fp32 O' the kernel blends
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    # o_hat vs the fp64 oracle, sampled rows (SSA from the explicit mask, then Eq. 3 in fp64)
    kf = gen_rows_f32(ks, 0, n)
    worst = 0.0
    for t in [0, 1, 127, 128, 383, 384, 700, 1023]:
        qr = gen_rows_f32(qs, t * H, H)
        osp, _ = oracle.attention_rows(qr, np.full(H, t), kf, kf[:, :D_V], SCALE, *PAT)
        ofr = gen_rows_f32(ofs, t * H, H)
        rh, _ = oracle.blend(ofr, osp, alpha)
        err = np.abs(oh[0, t].double().cpu().numpy().ravel() - rh).max()
        worst = max(worst, err)
    assert worst <= 2e-2, worst
    # d_alpha vs Eq. 3's gradient on the same bits: o_full, d_o_hat (bf16) and the fp32 O'
    f_of = of.float().cpu().numpy().ravel()
    f_dh = dh.float().cpu().numpy().ravel()
    f_os = o_sp32.cpu().numpy().ravel()
    _, rda = oracle.blend(f_of, f_os, alpha, f_dh)
    mag = float(np.abs(f_dh.astype(np.float64) * (f_of.astype(np.float64) - f_os)).sum())
    assert abs(float(da.item()) - rda) <= 1e-4 * mag, (float(da.item()), rda, mag)
    # deterministic: bitwise identical on repeat
    oh2, da2 = loza.ssa_prefill_blend(q, kv, of, _alpha(alpha), dh, pattern=PAT, scale=SCALE)
    torch.cuda.synchronize()
    assert torch.equal(oh2, oh) and float(da2.item()) == float(da.item())


def test_batched_ragged_paper_pattern():
    """batch 2, n = 1000 (ragged last unit), the paper's (1,7,128): alpha = 0.5 o_hat equals the unfused
    pipeline's fp32 evaluation within two bf16 roundings; d_alpha vs the oracle gradient."""
    n, B, pat = 1000, 2, (1, 7, 128)
    qs, ks, ofs, dhs = _inputs(23, n, B)
    q, kv, of, dh = (empty_filled(s) for s in (qs, ks, ofs, dhs))
    oh, da = loza.ssa_prefill_blend(q, kv, of, _alpha(0.5), dh, pattern=pat, scale=SCALE)
    o_sp32 = loza.ssa_prefill(q, kv, pattern=pat, scale=SCALE, out_dtype=torch.float32)
    torch.cuda.synchronize()
    ref = (0.5 * of.double() + 0.5 * o_sp32.double())
    assert (oh.double() - ref).abs().max().item() <= 2.0 ** -8 * ref.abs().max().item() + 1e-6
    f_of, f_dh, f_os = (x.float().cpu().numpy().ravel() for x in (of, dh, o_sp32))
    _, rda = oracle.blend(f_of, f_os, 0.5, f_dh)
    mag = float(np.abs(f_dh.astype(np.float64) * (f_of.astype(np.float64) - f_os)).sum())
    assert abs(float(da.item()) - rda) <= 1e-4 * mag


def test_bad_alpha_flags_status():
    n = 256
    qs, ks, ofs, dhs = _inputs(24, n)
    q, kv, of, dh = (empty_filled(s) for s in (qs, ks, ofs, dhs))
    for bad in (1.5, -0.1, float("nan")):
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _, da = loza.ssa_prefill_blend(q, kv, of, _alpha(bad), dh, pattern=PAT, scale=SCALE, status=st)
        torch.cuda.synchronize()
        assert int(st.item()) == 1 and np.isnan(float(da.item()))


def test_rejects_fp32_output():
    n = 256
    qs, ks, ofs, _ = _inputs(25, n)
    q, kv = empty_filled(qs), empty_filled(ks)
    of = torch.zeros((1, n, H, D_V), dtype=torch.float32, device="cuda")
    with pytest.raises((loza.LozaError, AssertionError)):
        loza.ssa_prefill_blend(q, kv, of, _alpha(0.5), pattern=PAT, scale=SCALE,
                               out=torch.empty((1, n, H, D_V), dtype=torch.float32, device="cuda"))


def test_d_alpha_end_to_end_vs_oracle_attention():
    """d_alpha of the fused kernel against Eq. 3's gradient on the ORACLE's own SSA output (fp64, explicit mask:
    PAPER.md:54-57), not on the kernel's O'. The two differ only through the attention error e = O'_kernel - O'_ref,
    so |d_alpha - d_alpha_ref| <= max|e| * sum|d_o_hat| (+ the 1e-4 summation allowance of DESIGN R12); max|e| is
    itself held to the bf16 attention tolerance 2e-2 (R12) on every row of the 512-token problem."""
    n, alpha = 512, 0.4
    qs, ks, ofs, dhs = _inputs(24, n)
    q, kv, of, dh = (empty_filled(s) for s in (qs, ks, ofs, dhs))
    oh, da = loza.ssa_prefill_blend(q, kv, of, _alpha(alpha), dh, pattern=PAT, scale=SCALE)
    torch.cuda.synchronize()
    qf = gen_rows_f32(qs, 0, n * H).reshape(1, n, H, D_QK)
    kf = gen_rows_f32(ks, 0, n).reshape(1, n, D_QK)
    o_ref, _ = oracle.attention(qf, kf, np.ascontiguousarray(kf[..., :D_V]), SCALE, pattern=PAT)
    o_sp32 = loza.ssa_prefill(q, kv, pattern=PAT, scale=SCALE, out_dtype=torch.float32)
    torch.cuda.synchronize()
    e = float(np.abs(o_sp32.double().cpu().numpy() - o_ref).max())
    assert e <= 2e-2, e
    f_of = gen_rows_f32(ofs, 0, n * H).ravel()
    f_dh = gen_rows_f32(dhs, 0, n * H).ravel()
    _, rda = oracle.blend(f_of, o_ref.ravel(), alpha, f_dh)
    sdh = float(np.abs(f_dh.astype(np.float64)).sum())
    mag = float(np.abs(f_dh.astype(np.float64) * (f_of.astype(np.float64) - o_ref.ravel())).sum())
    assert abs(float(da.item()) - rda) <= e * sdh + 1e-4 * mag, (float(da.item()), rda, e * sdh)
