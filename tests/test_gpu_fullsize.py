"""Parity at the BASELINE.json sizes the bench times, on sampled outputs the fp64 oracle computes one by one
(DESIGN.md §3): blend, the fused calibration forward and the backward at 8K (configs[2]), the ring-cache decode at position
1M (configs[3]), and the sequence-parallel prefill at 8 virtual ranks (the bench's largest topology).
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_DO, TID_K, TID_O_FULL, TID_O_SPARSE, TID_Q, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

H, D_QK, D_V = 64, 576, 512
PAT = (1, 7, 128)


def test_blend_8k_sampled():
    n = 8192
    mk = lambda tid: Spec(seed=51, tensor_id=tid, batch=1, n=n, heads=H, d=D_V)  # noqa: E731
    of, os_, dh = (empty_filled(mk(t)) for t in (TID_O_FULL, TID_O_SPARSE, TID_DO))
    a = torch.tensor([0.3], dtype=torch.float32, device="cuda")
    oh, da = loza.loza_blend(of.view(-1), os_.view(-1), a, dh.view(-1))
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    rows = rng.integers(0, n * H, 64)
    for r in rows:
        f = [gen_rows_f32(mk(t), int(r), 1)[0] for t in (TID_O_FULL, TID_O_SPARSE)]
        rh, _ = oracle.blend(f[0], f[1], 0.3)
        got = oh.view(n * H, D_V)[int(r)].double().cpu().numpy()
        assert np.abs(got - rh).max() <= 2.0 ** -8 * np.abs(rh).max() + 1e-6
    # d_alpha over the whole 268M elements: the oracle's Eq. 3 gradient (oracle.blend, fp64) on the same bits,
    # summed chunk by chunk on the host (the sum of the chunks' gradients is the gradient: Eq. 3 is linear)
    ref, mag = 0.0, 0.0
    for c in range(0, n, 512):
        f = [x[0, c:c + 512].float().cpu().numpy().ravel() for x in (of, os_, dh)]
        _, g = oracle.blend(f[0], f[1], 0.3, f[2])
        ref += g
        mag += float(np.abs(f[2].astype(np.float64) * (f[0].astype(np.float64) - f[1])).sum())
    assert abs(float(da.item()) - ref) <= 1e-4 * mag


def test_calibration_fused_8k_sampled():
    n = 8192
    qs = Spec(seed=52, tensor_id=TID_Q, batch=1, n=n, heads=H, d=D_QK)
    ks = Spec(seed=52, tensor_id=TID_K, batch=1, n=n, heads=1, d=D_QK)
    ofs = Spec(seed=52, tensor_id=TID_O_FULL, batch=1, n=n, heads=H, d=D_V)
    q, kv, of = empty_filled(qs), empty_filled(ks), empty_filled(ofs)
    a = torch.tensor([0.6], dtype=torch.float32, device="cuda")
    oh, _ = loza.ssa_prefill_blend(q, kv, of, a, pattern=PAT)
    torch.cuda.synchronize()
    kf = gen_rows_f32(ks, 0, n)
    scale = loza.default_scale(D_QK)
    for t in [0, 1023, 1024, 4097, 8191]:
        qr = gen_rows_f32(qs, t * H, H)
        osp, _ = oracle.attention_rows(qr, np.full(H, t), kf, kf[:, :D_V], scale, *PAT)
        rh, _ = oracle.blend(gen_rows_f32(ofs, t * H, H), osp, 0.6)
        assert np.abs(oh[0, t].double().cpu().numpy().ravel() - rh).max() <= 2e-2, t


def test_ring_decode_at_1m_sampled():
    """B = 8 sequences at absolute position 1,048,576 - 1 - j, ring caches filled from the windows'
    rows; rows against the oracle over the same window (sink block + 7 local blocks)."""
    B, T = 8, 1 << 20
    s, l, b = PAT
    ks = Spec(seed=53, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    qs = Spec(seed=53, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    q = empty_filled(qs)
    lens = [T - 7 * j for j in range(B)]
    cache = torch.zeros((B, (s + l) * b, D_QK), dtype=torch.bfloat16, device="cuda")
    for bi, L in enumerate(lens):
        # only the rows the window of position L-1 needs: the sink block and the last l blocks
        qb = (L - 1) // b
        starts = [0] + [k * b for k in range(max(s, qb - l + 1), qb + 1)]
        for st in starts:
            rows = torch.from_numpy(gen_rows_f32(ks, bi * T + st, min(b, L - st))).to("cuda").to(torch.bfloat16)
            loza.ssa_ring_append(cache[bi:bi + 1], rows.unsqueeze(0),
                                 torch.tensor([st], dtype=torch.int32, device="cuda"), pattern=PAT)
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    o = loza.ssa_decode_ring(q, cache, seq, pattern=PAT)
    torch.cuda.synchronize()
    scale = loza.default_scale(D_QK)
    for bi, L in enumerate(lens):
        keys = oracle.allowed_keys(L - 1, L, s, l, b)
        kf = np.stack([gen_rows_f32(ks, bi * T + int(j), 1)[0] for j in keys])
        qr = gen_rows_f32(qs, bi * H, H)
        ref, _ = oracle.attend(qr, kf, kf[:, :D_V], scale)
        assert np.abs(o[bi, 0].double().cpu().numpy() - ref).max() <= 2e-2, bi


def test_seqpar_8_virtual_ranks_bitwise():
    """8 ranks x 4096 tokens (32K total, MLA bf16, (1,7,128)): every shard through the exchange-then-SSA path
    equals the single-GPU prefill bitwise."""
    world, n_local = 8, 4096
    n = world * n_local
    qs = Spec(seed=54, tensor_id=TID_Q, batch=1, n=n, heads=H, d=D_QK)
    ks = Spec(seed=54, tensor_id=TID_K, batch=1, n=n, heads=1, d=D_QK)
    q, kv = empty_filled(qs), empty_filled(ks)
    ref = loza.ssa_prefill(q, kv, pattern=PAT)
    shards = [kv[:, r * n_local:(r + 1) * n_local].contiguous() for r in range(world)]
    for r in range(world):
        o = loza.ssa_seqpar_prefill_local(q[:, r * n_local:(r + 1) * n_local].contiguous(), shards[r], None, PAT,
                                          loza.default_scale(D_QK), rank=r, world=world, rank0_k=shards[0],
                                          prev_k=shards[r - 1] if r > 0 else None)
        torch.cuda.synchronize()
        assert torch.equal(o, ref[:, r * n_local:(r + 1) * n_local]), r


def test_mha_prefill_32k_sampled():
    """MHA-form SSA prefill at the bench shape: B1, 32768 tokens, H64, q/k 192, v 128,
    (1,7,128); sampled (token, head) rows against the oracle over the token's window."""
    from inputs import TID_V
    n, Hm = 32768, 64
    specs = [Spec(seed=55, tensor_id=t, batch=1, n=n, heads=Hm, d=d) for t, d in ((TID_Q, 192), (TID_K, 192), (TID_V, 128))]
    q, k, v = (empty_filled(s, four_d=True) for s in specs)
    o = loza.ssa_prefill_mha(q, k, v, PAT)
    torch.cuda.synchronize()
    s, l, b = PAT
    scale = 1.0 / np.sqrt(192.0)
    for t, h in [(0, 0), (127, 5), (1023, 63), (1024, 17), (20000, 31), (32767, 2)]:
        keys = oracle.allowed_keys(t, n, s, l, b)
        kb = sorted({int(j) // b for j in keys})
        kk = np.concatenate([gen_rows_f32(specs[1], blk * b * Hm, b * Hm).reshape(b, Hm, 192)[:, h] for blk in kb])
        vv = np.concatenate([gen_rows_f32(specs[2], blk * b * Hm, b * Hm).reshape(b, Hm, 128)[:, h] for blk in kb])
        pos = np.concatenate([np.arange(blk * b, blk * b + b) for blk in kb])
        sel = np.isin(pos, keys)
        qr = gen_rows_f32(specs[0], t * Hm + h, 1)
        ref, _ = oracle.attend(qr, kk[sel], vv[sel], scale)
        assert np.abs(o[0, t, h].double().cpu().numpy() - ref[0]).max() <= 2e-2, (t, h)


def test_backward_8k_sampled():
    """Attention backward (the tensor-core kernels) at the bench shape: B1, 8192 tokens, H64,
    MLA 576/512, (1,7,128), bf16, in the bench's launch configuration.
    - dQ of sampled (token, head) rows against the oracle backward over those rows (a dQ row depends on its
      own row only);
    - dK, dV of the last 8 keys against the oracle backward over the 512 rows that attend them (causal);
    - at full size, two identities of the gradient: sum_j dS_rj = 0 for every row (so sum_j dK_j = 0) and
      sum_j P_rj = 1 (so sum_j dV_j = sum_r dO_r). They cover every key, the sink tiles and their split
      reduction included. Tolerance: each dK_j / dV_j may carry a bf16-operand rounding error of relative
      size 2^-7 in an independent direction, so the sums may deviate by 2^-7 * sqrt(sum_j ||.||^2); a dropped
      term or a lost split is orders of magnitude larger."""
    n = 8192
    qs = Spec(seed=56, tensor_id=TID_Q, batch=1, n=n, heads=H, d=D_QK)
    ks = Spec(seed=56, tensor_id=TID_K, batch=1, n=n, heads=1, d=D_QK)
    ds = Spec(seed=56, tensor_id=TID_DO, batch=1, n=n, heads=H, d=D_V)
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(ds)
    scale = loza.default_scale(D_QK)
    lse = torch.empty((1, H, n), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=PAT, scale=scale, lse=lse)
    dq, dk, dv = loza.attention_backward(q, kv, o, lse, do, pattern=PAT, scale=scale)
    torch.cuda.synchronize()
    kf = gen_rows_f32(ks, 0, n)
    samples = [(0, 0), (127, 9), (128, 63), (1000, 1), (1023, 40), (1024, 7), (5000, 33), (8191, 62)]
    qr = np.concatenate([gen_rows_f32(qs, t * H + h, 1) for t, h in samples])
    dr = np.concatenate([gen_rows_f32(ds, t * H + h, 1) for t, h in samples])
    rq, _, _ = oracle.attention_backward(qr, np.array([t for t, _ in samples]), kf, kf[:, :D_V], dr, scale, *PAT)
    got = np.stack([dq[0, t, h].double().cpu().numpy() for t, h in samples])
    assert np.abs(got - rq).max() / np.abs(rq).max() <= 2e-2
    t0 = n - 8
    _, rk, rv = oracle.attention_backward(gen_rows_f32(qs, t0 * H, 8 * H), np.repeat(np.arange(t0, n), H), kf,
                                          kf[:, :D_V], gen_rows_f32(ds, t0 * H, 8 * H), scale, *PAT)
    assert np.abs(dk[0, t0:].double().cpu().numpy() - rk[t0:]).max() / np.abs(rk[t0:]).max() <= 2e-2
    assert np.abs(dv[0, t0:].double().cpu().numpy() - rv[t0:]).max() / np.abs(rv[t0:]).max() <= 2e-2
    dk64, dv64 = dk[0].double(), dv[0].double()
    assert dk64.sum(0).norm().item() <= 2.0 ** -7 * dk64.pow(2).sum().sqrt().item()
    sd = do[0].double().reshape(-1, D_V).sum(0)
    assert (dv64.sum(0) - sd).norm().item() <= 2.0 ** -7 * dv64.pow(2).sum().sqrt().item()
