"""GPU parity: generator twin, block selection, fp32 SIMT attention (tiny config), blend + d_alpha.

All through the C ABI (paper_2512_23966_b200.loza); expected values from oracle/ only.
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_DO, TID_K, TID_O_FULL, TID_O_SPARSE, TID_Q, TID_V, Spec, gen_rows_bits, gen_rows_f32
from inputs.device import empty_filled, fill_
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu

TINY = dict(n=1024, H=1, d=64, s=1, l=2, b=64, scale=1.0 / 8.0)  # BASELINE.json configs[0]


def _normwise(gpu, ref):
    return float(np.abs(gpu - ref).max() / np.abs(ref).max())


@pytest.mark.parametrize("kind", ["plain", "kv_marker", "kv_sink", "q_sink"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_generator_twin_bitwise(kind, dtype):
    sp = Spec(seed=7, tensor_id=TID_K, batch=2, n=300, heads=3, d=40, dtype=dtype, kind=kind, block=16,
              marker_mod=32, amp=0.5, col=5, sink_rows=16)
    t = empty_filled(sp)
    host = gen_rows_bits(sp, 0, sp.rows).reshape(-1)
    dev = t.view(torch.int16 if dtype == "bf16" else torch.int32).cpu().numpy().reshape(-1)
    assert np.array_equal(dev.view(np.uint16 if dtype == "bf16" else np.float32).view(np.uint8),
                          host.view(np.uint8))
    part = torch.empty(50 * sp.d, dtype=t.dtype, device="cuda")
    fill_(part, sp, row_start=123)
    assert torch.equal(part.view(-1), t.view(-1)[123 * sp.d:173 * sp.d])


@pytest.mark.parametrize("pattern", [(1, 7, 128), (1, 2, 64), (0, 1, 1), (3, 2, 5), (2, 9, 16)])
@pytest.mark.parametrize("n,q_start", [(1, 0), (1000, 0), (4096, 0), (777, 0)])
def test_select_blocks_bit_exact(pattern, n, q_start):
    s, l, b = pattern
    idx, cnt = loza.ssa_select_blocks(n, q_start, pattern)
    ridx, rcnt = oracle.select_blocks(n, q_start, q_start + n, s, l, b)
    assert np.array_equal(cnt.cpu().numpy(), rcnt)
    assert np.array_equal(idx.cpu().numpy(), ridx)


def test_select_blocks_q_start_and_large():
    s, l, b = 1, 7, 128
    idx, cnt = loza.ssa_select_blocks(1 << 20, 0, (s, l, b))
    qbs = np.array([0, 1, 6, 7, 8, 4095, 8191])
    ridx, rcnt = oracle.select_blocks(1 << 20, 0, 1 << 20, s, l, b, qb_list=qbs)
    assert np.array_equal(idx.cpu().numpy()[qbs], ridx) and np.array_equal(cnt.cpu().numpy()[qbs], rcnt)
    idx2, cnt2 = loza.ssa_select_blocks(4096, 8192, (s, l, b))
    r2, c2 = oracle.select_blocks(4096, 8192, 8192 + 4096, s, l, b)
    assert np.array_equal(idx2.cpu().numpy(), r2) and np.array_equal(cnt2.cpu().numpy(), c2)


def _tiny_inputs(seed, kind="plain", B=1, n=None, H=None, d=None):
    c = TINY
    n = n or c["n"]
    H = H or c["H"]
    d = d or c["d"]
    qs = Spec(seed=seed, tensor_id=TID_Q, batch=B, n=n, heads=H, d=d, dtype="f32",
              kind="q_sink" if kind == "sink" else "plain", amp=5.27, col=d - 1)
    ks = Spec(seed=seed, tensor_id=TID_K, batch=B, n=n, heads=1, d=d, dtype="f32",
              kind="kv_sink" if kind == "sink" else "plain", amp=5.27, col=d - 1, sink_rows=c["b"])
    vs = Spec(seed=seed, tensor_id=TID_V, batch=B, n=n, heads=1, d=d, dtype="f32",
              kind="kv_marker" if kind == "marker" else "plain", block=c["b"], marker_mod=d, amp=0.5)
    return qs, ks, vs


@pytest.mark.parametrize("seed,kind", [(0, "plain"), (1, "marker"), (2, "sink")])
@pytest.mark.parametrize("mode", ["ssa", "full"])
def test_tiny_fp32_prefill_vs_oracle(seed, kind, mode):
    c = TINY
    qs, ks, vs = _tiny_inputs(seed, kind)
    q, k, v = empty_filled(qs), empty_filled(ks), empty_filled(vs)
    lse = torch.empty((1, 1, c["n"]), device="cuda", dtype=torch.float32)
    if mode == "ssa":
        o = loza.ssa_prefill(q, k, v, (c["s"], c["l"], c["b"]), c["scale"], lse=lse)
    else:
        o = loza.full_attn_ref(q, k, v, c["scale"], lse=lse)
    torch.cuda.synchronize()
    qf = gen_rows_f32(qs, 0, qs.rows)
    kf, vf = gen_rows_f32(ks, 0, ks.rows), gen_rows_f32(vs, 0, vs.rows)
    ref, rlse = oracle.attention_rows(qf, np.arange(c["n"]), kf, vf, c["scale"], c["s"], c["l"], c["b"],
                                      sparse=(mode == "ssa"))
    got = o[0, :, 0].double().cpu().numpy()
    assert _normwise(got, ref) <= 1e-4
    assert np.abs(lse[0, 0].double().cpu().numpy() - rlse).max() <= 1e-4 * np.abs(rlse).max()


def test_tiny_fp32_batched_multihead_and_q_start():
    s, l, b, n, H, d = 1, 3, 16, 200, 4, 32
    qs = Spec(seed=5, tensor_id=TID_Q, batch=2, n=n, heads=H, d=d, dtype="f32")
    ks = Spec(seed=5, tensor_id=TID_K, batch=2, n=n, heads=1, d=d, dtype="f32")
    vs = Spec(seed=5, tensor_id=TID_V, batch=2, n=n, heads=1, d=24, dtype="f32")
    q, k, v = empty_filled(qs), empty_filled(ks), empty_filled(vs)
    q_start = 64
    o = loza.ssa_prefill(q[:, q_start:], k, v, (s, l, b), 0.3, q_start=q_start)
    torch.cuda.synchronize()
    for bi in range(2):
        qf = gen_rows_f32(qs, (bi * n + q_start) * H, (n - q_start) * H)
        kf, vf = gen_rows_f32(ks, bi * n, n), gen_rows_f32(vs, bi * n, n)
        pos = np.repeat(np.arange(q_start, n), H)
        ref, _ = oracle.attention_rows(qf, pos, kf, vf, 0.3, s, l, b)
        assert _normwise(o[bi].reshape(-1, 24).double().cpu().numpy(), ref) <= 1e-4


def test_tiny_fp32_decode_vs_oracle_and_prefill():
    c = TINY
    B, n = 3, c["n"]
    qs, ks, vs = _tiny_inputs(3, B=B)
    q, k, v = empty_filled(qs), empty_filled(ks), empty_filled(vs)
    seq = torch.tensor([1, 513, 1024], dtype=torch.int32, device="cuda")
    qd = torch.stack([q[i, seq[i] - 1] for i in range(B)])[:, None]  # [B,1,H,d]
    pat = (c["s"], c["l"], c["b"])
    od = loza.ssa_decode(qd, k, seq, v, pat, c["scale"])
    of = loza.full_attn_ref(qd, k, v, c["scale"], seq_lens=seq)
    op = loza.ssa_prefill(q, k, v, pat, c["scale"])
    torch.cuda.synchronize()
    for i, t in enumerate(seq.tolist()):
        kf, vf = gen_rows_f32(ks, i * n, t), gen_rows_f32(vs, i * n, t)
        qf = gen_rows_f32(qs, i * n + t - 1, 1)
        ref, _ = oracle.attention_rows(qf, [t - 1], kf, vf, c["scale"], *pat)
        reff, _ = oracle.attention_rows(qf, [t - 1], kf, vf, c["scale"], sparse=False)
        assert _normwise(od[i, 0].double().cpu().numpy(), ref) <= 1e-4
        assert _normwise(of[i, 0].double().cpu().numpy(), reff) <= 1e-4
        # streaming equivalence: decode at t == row t-1 of the prefill, same kernel arithmetic
        assert torch.allclose(od[i, 0], op[i, t - 1], atol=1e-6, rtol=0)


def test_tiny_fp32_closed_forms_on_gpu():
    n, d = 64, 16
    qs = Spec(seed=9, tensor_id=TID_Q, batch=1, n=n, heads=1, d=d, dtype="f32")
    vs = Spec(seed=9, tensor_id=TID_V, batch=1, n=n, heads=1, d=d, dtype="f32")
    q, v = empty_filled(qs), empty_filled(vs)
    # (s=0, l=1, b=1): O = V
    o = loza.ssa_prefill(q, q[:, :, 0], v, (0, 1, 1), 0.5)
    torch.cuda.synchronize()
    assert torch.equal(o[0, :, 0], v[0])
    # V == c => O == c
    c = torch.full_like(v, 0.375)
    o2 = loza.ssa_prefill(q, q[:, :, 0], c, (1, 1, 8), 0.5)
    torch.cuda.synchronize()
    assert float((o2 - 0.375).abs().max()) < 1e-6


@pytest.mark.parametrize("world", [2, 4])
def test_seqpar_local_emulation_matches_single_gpu(world):
    s, l, b, H, d = 1, 3, 16, 2, 32
    n = 64 * world
    qs = Spec(seed=11, tensor_id=TID_Q, batch=2, n=n, heads=H, d=d, dtype="f32")
    ks = Spec(seed=11, tensor_id=TID_K, batch=2, n=n, heads=1, d=d, dtype="f32")
    q, kv = empty_filled(qs), empty_filled(ks)
    ref = loza.ssa_prefill(q, kv, kv[..., :24], (s, l, b), 0.2, d_v=24)
    nl = n // world
    shards_k = [kv[:, r * nl:(r + 1) * nl].contiguous() for r in range(world)]
    for r in range(world):
        o = loza.ssa_seqpar_prefill_local(q[:, r * nl:(r + 1) * nl].contiguous(), shards_k[r], None, (s, l, b), 0.2,
                                          rank=r, world=world, rank0_k=shards_k[0],
                                          prev_k=shards_k[r - 1] if r > 0 else None, d_v=24)
        torch.cuda.synchronize()
        assert torch.equal(o, ref[:, r * nl:(r + 1) * nl]), r


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("alpha", [0.0, 0.25, 0.5, 1.0])
def test_blend_vs_oracle(dtype, alpha):
    numel = 64 * 1024 + 8
    mk = lambda tid: Spec(seed=1, tensor_id=tid, batch=1, n=numel // 8, heads=1, d=8, dtype=dtype)  # noqa: E731
    of, os_, dh = (empty_filled(mk(t)).view(-1) for t in (TID_O_FULL, TID_O_SPARSE, TID_DO))
    a = torch.tensor([alpha], dtype=torch.float32, device="cuda")
    st = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    oh, da = loza.loza_blend(of, os_, a, dh, status=st)
    torch.cuda.synchronize()
    f = [gen_rows_f32(mk(t), 0, numel // 8).reshape(-1) for t in (TID_O_FULL, TID_O_SPARSE, TID_DO)]
    rh, rda = oracle.blend(f[0], f[1], alpha, f[2])
    got = oh.double().cpu().numpy()
    # fp32 evaluation: fma(a, x, (1-a)*y) -> <= ~2 fp32 roundings of |a x| + |(1-a) y|; bf16 output adds half an ulp
    mag_terms = alpha * np.abs(f[0].astype(np.float64)) + (1 - alpha) * np.abs(f[1].astype(np.float64))
    tol = 2.0 ** -21 * mag_terms + (2.0 ** -8 * np.abs(rh) if dtype == "bf16" else 0.0)
    assert (np.abs(got - rh) <= tol).all()
    if alpha == 1.0:
        assert torch.equal(oh, of)
    if alpha == 0.0:
        assert torch.equal(oh, os_)
    mag = float(np.abs(f[2].astype(np.float64) * (f[0].astype(np.float64) - f[1])).sum())
    assert abs(float(da.item()) - rda) <= 1e-4 * mag
    assert int(st.item()) == 0
    # determinism: bitwise identical on repeat
    _, da2 = loza.loza_blend(of, os_, a, dh, want_out=False)
    torch.cuda.synchronize()
    assert float(da2.item()) == float(da.item())


def test_blend_bad_alpha_flags_status():
    x = torch.zeros(64, dtype=torch.bfloat16, device="cuda")
    for bad in (1.5, -0.1, float("nan")):
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _, da = loza.loza_blend(x, x, torch.tensor([bad], device="cuda"), x, status=st)
        torch.cuda.synchronize()
        assert int(st.item()) == 1 and np.isnan(float(da.item()))
