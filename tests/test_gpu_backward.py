"""GPU parity of attention_backward against the fp64 oracle backward (itself pinned by
finite differences of the forward oracle, tests/test_oracle_pins.py).

Tolerances (R12): fp32 inputs normwise ||d||_inf / ||ref||_inf <= 1e-4; bf16 MLA <= 2e-2 (the
forward's O, used for D = dO . O, is bf16-rounded: ~2^-9 relative, and P is recomputed from the forward LSE).
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_DO, TID_K, TID_Q, TID_V, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu


def _norm_err(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


@pytest.mark.parametrize("sparse", [True, False])
def test_backward_tiny_fp32(sparse):
    """configs[0] shape (H=1, d=64, separate K/V, fp32), all rows and keys."""
    B, n, H, d = 1, 512, 1, 64
    pat = (1, 2, 64)
    qs = Spec(seed=41, tensor_id=TID_Q, batch=B, n=n, heads=H, d=d, dtype="f32")
    ks = Spec(seed=41, tensor_id=TID_K, batch=B, n=n, heads=1, d=d, dtype="f32")
    vs = Spec(seed=41, tensor_id=TID_V, batch=B, n=n, heads=1, d=d, dtype="f32")
    ds = Spec(seed=41, tensor_id=TID_DO, batch=B, n=n, heads=H, d=d, dtype="f32")
    q, k, v, do = (empty_filled(s) for s in (qs, ks, vs, ds))
    scale = 0.125
    lse = torch.empty((B, H, n), device="cuda")
    if sparse:
        o = loza.ssa_prefill(q, k, v, pat, scale, d_v=d, lse=lse)
    else:
        o = loza.full_attn_ref(q, k, v, scale, d_v=d, lse=lse)
    dq, dk, dv = loza.attention_backward(q, k, o, lse, do, v=v, pattern=pat if sparse else None, scale=scale, d_v=d)
    torch.cuda.synchronize()
    rq, rk, rv = oracle.attention_backward(gen_rows_f32(qs, 0, n), np.arange(n), gen_rows_f32(ks, 0, n),
                                           gen_rows_f32(vs, 0, n), gen_rows_f32(ds, 0, n), scale, *pat,
                                           sparse=sparse)
    assert _norm_err(dq[0, :, 0].double().cpu().numpy(), rq) <= 1e-4
    assert _norm_err(dk[0].double().cpu().numpy(), rk) <= 1e-4
    assert _norm_err(dv[0].double().cpu().numpy(), rv) <= 1e-4


def test_backward_mla_bf16_ssa():
    """absorbed MLA shape (576/512, H=64, V = KV[:, :512]), bf16, (1,1,128) over n = 256 (a sink-only and a
    sink+local query block), every row and key; MLA cache gradient d_kv = d_k + [d_v, 0]."""
    B, n, H = 1, 256, 64
    pat = (1, 1, 128)
    qs = Spec(seed=42, tensor_id=TID_Q, batch=B, n=n, heads=H, d=576)
    ks = Spec(seed=42, tensor_id=TID_K, batch=B, n=n, heads=1, d=576)
    ds = Spec(seed=42, tensor_id=TID_DO, batch=B, n=n, heads=H, d=512)
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(ds)
    scale = loza.default_scale(576)
    lse = torch.empty((B, H, n), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=scale, lse=lse)
    dq, dk, dv = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
    dq2, dk2, dv2 = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
    torch.cuda.synchronize()
    assert torch.equal(dq, dq2) and torch.equal(dk, dk2) and torch.equal(dv, dv2)  # deterministic
    kf = gen_rows_f32(ks, 0, n)
    rq, rk, rv = oracle.attention_backward(gen_rows_f32(qs, 0, n * H), np.repeat(np.arange(n), H), kf, kf[:, :512],
                                           gen_rows_f32(ds, 0, n * H), scale, *pat)
    assert _norm_err(dq[0].reshape(n * H, 576).double().cpu().numpy(), rq) <= 2e-2
    assert _norm_err(dk[0].double().cpu().numpy(), rk) <= 2e-2
    assert _norm_err(dv[0].double().cpu().numpy(), rv) <= 2e-2
    # MLA: the cache gradient composes d_k and d_v
    dkv = dk.clone()
    dkv[..., :512] += dv
    rkv = rk.copy()
    rkv[:, :512] += rv
    assert _norm_err(dkv[0].double().cpu().numpy(), rkv) <= 2e-2


def test_backward_q_start_offset():
    """queries [q_start, n) against keys [0, n) (chunked prefill), fp32 tiny dims, SSA."""
    B, n, H, d, q0 = 1, 384, 2, 32, 128
    pat = (1, 2, 64)
    qs = Spec(seed=43, tensor_id=TID_Q, batch=B, n=n, heads=H, d=d, dtype="f32")
    ks = Spec(seed=43, tensor_id=TID_K, batch=B, n=n, heads=1, d=d, dtype="f32")
    ds = Spec(seed=43, tensor_id=TID_DO, batch=B, n=n, heads=H, d=d, dtype="f32")
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(ds)
    scale = 0.2
    lse = torch.empty((B, H, n - q0), device="cuda")
    qq = q[:, q0:].contiguous()
    dd = do[:, q0:].contiguous()
    o = loza.ssa_prefill(qq, kv, kv, pat, scale, d_v=d, q_start=q0, lse=lse)
    dq, dk, dv = loza.attention_backward(qq, kv, o, lse, dd, v=kv, pattern=pat, scale=scale, d_v=d, q_start=q0)
    torch.cuda.synchronize()
    kf = gen_rows_f32(ks, 0, n)
    rq, rk, rv = oracle.attention_backward(gen_rows_f32(qs, q0 * H, (n - q0) * H), np.repeat(np.arange(q0, n), H),
                                           kf, kf, gen_rows_f32(ds, q0 * H, (n - q0) * H), scale, *pat)
    assert _norm_err(dq[0].reshape(-1, d).double().cpu().numpy(), rq) <= 1e-4
    assert _norm_err(dk[0].double().cpu().numpy(), rk) <= 1e-4
    assert _norm_err(dv[0].double().cpu().numpy(), rv) <= 1e-4


@pytest.mark.parametrize("sparse,causal,q0", [(True, True, 0), (False, True, 0), (False, False, 0), (True, True, 128)])
def test_backward_tiled_fp32_h8(sparse, causal, q0):
    """The tiled backward kernels (H % 8 == 0, b % 16 == 0): fp32, H = 8, separate K / V, d 64 / 48, every row
    and key against the fp64 oracle backward (1e-4 normwise)."""
    B, n, H, dq_, dv_ = 2, 640, 8, 64, 48
    pat = (1, 2, 64)
    qs = Spec(seed=44, tensor_id=TID_Q, batch=B, n=n, heads=H, d=dq_, dtype="f32")
    ks = Spec(seed=44, tensor_id=TID_K, batch=B, n=n, heads=1, d=dq_, dtype="f32")
    vs = Spec(seed=44, tensor_id=TID_V, batch=B, n=n, heads=1, d=dv_, dtype="f32")
    ds = Spec(seed=44, tensor_id=TID_DO, batch=B, n=n, heads=H, d=dv_, dtype="f32")
    q, k, v, do = (empty_filled(s) for s in (qs, ks, vs, ds))
    qq, dd = q[:, q0:].contiguous(), do[:, q0:].contiguous()
    scale = 0.11
    lse = torch.empty((B, H, n - q0), device="cuda")
    if sparse:
        o = loza.ssa_prefill(qq, k, v, pat, scale, d_v=dv_, lse=lse, q_start=q0)
    else:
        o = loza.full_attn_ref(qq, k, v, scale, d_v=dv_, lse=lse, causal=causal, q_start=q0)
    dq, dk, dv = loza.attention_backward(qq, k, o, lse, dd, v=v, pattern=pat if sparse else None, scale=scale,
                                         d_v=dv_, causal=causal, q_start=q0)
    torch.cuda.synchronize()
    for bi in range(B):
        rq, rk, rv = oracle.attention_backward(gen_rows_f32(qs, (bi * n + q0) * H, (n - q0) * H),
                                               np.repeat(np.arange(q0, n), H), gen_rows_f32(ks, bi * n, n),
                                               gen_rows_f32(vs, bi * n, n), gen_rows_f32(ds, (bi * n + q0) * H, (n - q0) * H),
                                               scale, *pat, sparse=sparse, causal=causal)
        assert _norm_err(dq[bi].reshape(-1, dq_).double().cpu().numpy(), rq) <= 1e-4
        assert _norm_err(dk[bi].double().cpu().numpy(), rk) <= 1e-4
        assert _norm_err(dv[bi].double().cpu().numpy(), rv) <= 1e-4


@pytest.mark.parametrize("sparse,causal,q0,H,n,pat,B,ofwd", [
    (True, True, 0, 16, 640, (1, 2, 128), 2, False),    # 4 tokens per 64-row tile, 3 sink splits
    (True, True, 0, 8, 1152, (1, 7, 128), 1, False),    # the paper's pattern, a window boundary inside the sequence
    (True, True, 128, 8, 512, (1, 2, 128), 1, False),   # chunked prefill (q_start)
    (True, True, 0, 64, 400, (2, 1, 128), 1, False),    # two sink blocks, H = 64, ragged last block
    (False, True, 0, 8, 304, None, 1, False),           # full causal, ragged key tile
    (False, False, 0, 8, 208, None, 1, False),          # bidirectional
    (True, True, 0, 8, 300, (1, 1, 128), 1, True),      # ragged row tile (2400 rows), 3 sink splits
    (False, True, 0, 8, 100, None, 1, True),            # ragged rows and keys, one partial key tile set
    (True, True, 0, 24, 300, (1, 1, 128), 1, True),     # H = 24: tcgen05 keys, dQ by the warp-MMA row kernel
    (True, True, 0, 128, 300, (1, 1, 128), 1, True),    # H = 128: one token per 128-row dQ tile
    (True, True, 0, 8, 400, (0, 2, 128), 1, True),      # no sink blocks (s = 0): no sink tiles or splits
    (True, True, 0, 16, 1280, (1, 2, 256), 1, False),   # b = 256: 8 key tiles per block, 2 splits
])
def test_backward_mla_mma(sparse, causal, q0, H, n, pat, B, ofwd):
    """The tensor-core backward (SSA: D, tcgen05 key kernels writing dS rows -- the 128-key CTA-pair kernels when
    b = 128, 64-key kernels otherwise -- and tcgen05 dQ = dS K; full attention:
    the attn_bwd_mma.cu row kernel + tcgen05 key kernel; bf16, 576/512, V = KV[:, :512]) against the fp64 oracle
    backward, every row and key, bf16 tolerance (2e-2 normwise); deterministic across calls. ofwd: O and LSE
    from the oracle forward (rounded to bf16 / fp32), for row counts the bf16 forward does not take."""
    qs = Spec(seed=45, tensor_id=TID_Q, batch=B, n=n, heads=H, d=576)
    ks = Spec(seed=45, tensor_id=TID_K, batch=B, n=n, heads=1, d=576)
    ds = Spec(seed=45, tensor_id=TID_DO, batch=B, n=n, heads=H, d=512)
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(ds)
    qq, dd = q[:, q0:].contiguous(), do[:, q0:].contiguous()
    scale = loza.default_scale(576)
    lse = torch.empty((B, H, n - q0), device="cuda")
    if ofwd:
        o = torch.empty((B, n - q0, H, 512), dtype=torch.bfloat16, device="cuda")
        for bi in range(B):
            kf = gen_rows_f32(ks, bi * n, n)
            orow, lrow = oracle.attention_rows(gen_rows_f32(qs, (bi * n + q0) * H, (n - q0) * H),
                                               np.repeat(np.arange(q0, n), H), kf, kf[:, :512], scale,
                                               *(pat or (0, 1, 1)), sparse=sparse, causal=causal)
            o[bi] = torch.from_numpy(orow.reshape(n - q0, H, 512)).to(torch.bfloat16)
            lse[bi] = torch.from_numpy(lrow.reshape(n - q0, H).T.copy()).float()
    elif sparse:
        o = loza.ssa_prefill(qq, kv, pattern=pat, scale=scale, lse=lse, q_start=q0)
    else:
        o = loza.full_attn_ref(qq, kv, scale=scale, lse=lse, causal=causal, q_start=q0)
    run = lambda: loza.attention_backward(qq, kv, o, lse, dd, pattern=pat if sparse else None, scale=scale,  # noqa: E731
                                          causal=causal, q_start=q0)
    dq, dk, dv = run()
    dq2, dk2, dv2 = run()
    torch.cuda.synchronize()
    assert torch.equal(dq, dq2) and torch.equal(dk, dk2) and torch.equal(dv, dv2)
    for bi in range(B):
        kf = gen_rows_f32(ks, bi * n, n)
        rq, rk, rv = oracle.attention_backward(gen_rows_f32(qs, (bi * n + q0) * H, (n - q0) * H),
                                               np.repeat(np.arange(q0, n), H), kf, kf[:, :512],
                                               gen_rows_f32(ds, (bi * n + q0) * H, (n - q0) * H), scale,
                                               *(pat or (0, 1, 1)), sparse=sparse, causal=causal)
        assert _norm_err(dq[bi].reshape(-1, 576).double().cpu().numpy(), rq) <= 2e-2
        assert _norm_err(dk[bi].double().cpu().numpy(), rk) <= 2e-2
        assert _norm_err(dv[bi].double().cpu().numpy(), rv) <= 2e-2


def test_backward_mla_simt_forced():
    """The FFMA kernels stay reachable for the MLA shape (test knob backward = 1, loza_debug_force_kernel, set by
    tests/conftest.py from LOZA_TEST_BACKWARD_KERNEL): the bf16 MLA test through them."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_backward.py") + "::test_backward_mla_bf16_ssa"],
                       cwd=root, env=dict(os.environ, LOZA_TEST_BACKWARD_KERNEL="1"), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"LOZA_TEST_BACKWARD_KERNEL": "2"}, {"LOZA_TEST_BACKWARD_KERNEL": "3"},
                                 {"LOZA_TEST_BACKWARD_KERNEL": "4"}, {"LOZA_TEST_BACKWARD_KERNEL": "5"}])
def test_backward_mma_paths_forced(env):
    """The other key / dQ kernels kept reachable through the MLA parity cases (test knob backward,
    loza_debug_force_kernel): 2 = the warp-MMA key kernel and row kernel of attn_bwd_mma.cu instead of the
    tcgen05 key kernels and dS GEMM; 3 = tcgen05 key kernels, dQ by the row kernel instead of the tcgen05 dS
    GEMM; 4 = the 32-key tcgen05 key kernel (dK and dV in one pass) instead of the 64-key dV / dK pair; 5 = the
    64-key dV / dK kernels where the 128-key CTA-pair kernels are the default (SSA, b = 128)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", "-k", "mla",
                        os.path.join(root, "tests", "test_gpu_backward.py")],
                       cwd=root, env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_backward_graph_capture_bitwise():
    """The SSA backward (D on a side stream joined back before the dK kernel, the 64-key dV / dK kernels, the dS
    GEMM) captured in a CUDA graph and replayed equals the eager call bit for bit (it is deterministic)."""
    B, n, H = 1, 512, 64
    pat = (1, 2, 128)
    qs = Spec(seed=61, tensor_id=TID_Q, batch=B, n=n, heads=H, d=576)
    ks = Spec(seed=61, tensor_id=TID_K, batch=B, n=n, heads=1, d=576)
    ds = Spec(seed=61, tensor_id=TID_DO, batch=B, n=n, heads=H, d=512)
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(ds)
    scale = loza.default_scale(576)
    lse = torch.empty((B, H, n), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=scale, lse=lse)
    ref = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            out = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(out, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("n,H,B,keys", [(2048, 8, 1, (5, 700, 1900)), (4096, 8, 1, (1300, 4000)),
                                         (1024, 8, 3, (5, 900)), (4096, 64, 1, ())])
def test_backward_pair_splits_repeat_bitwise(n, H, B, keys):
    """The 128-key CTA-pair key kernels with their row splits (short sequences: every tile cut into query-block
    pieces, partials summed by a fixed-order reduce) and the pair dQ GEMM: five calls give the
    same bits (cross-CTA exchanges, DSMEM copies and partial reduces are ordered), and the dK / dV rows of
    sampled keys -- a sink key, keys of early and late local blocks -- match the fp64 oracle backward over every
    row that attends them (2e-2 normwise)."""
    pat = (1, 7, 128)
    qs = Spec(seed=71, tensor_id=TID_Q, batch=B, n=n, heads=H, d=576)
    ks = Spec(seed=71, tensor_id=TID_K, batch=B, n=n, heads=1, d=576)
    ds = Spec(seed=71, tensor_id=TID_DO, batch=B, n=n, heads=H, d=512)
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(ds)
    scale = loza.default_scale(576)
    lse = torch.empty((B, H, n), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=pat, scale=scale, lse=lse)
    ref = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
    for _ in range(4):
        out = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
        for a, b in zip(out, ref):
            assert torch.equal(a, b)
    _, dk, dv = ref
    bi = B - 1
    kf = gen_rows_f32(ks, bi * n, n)
    for j in keys:  # rows attending key j: tokens j .. the end of its window (every token for a sink key)
        t_hi = n if j < 128 else min(n, (j // 128 + 7) * 128)
        toks = np.arange(j, t_hi)
        _, rk, rv = oracle.attention_backward(gen_rows_f32(qs, (bi * n + j) * H, (t_hi - j) * H),
                                              np.repeat(toks, H), kf, kf[:, :512],
                                              gen_rows_f32(ds, (bi * n + j) * H, (t_hi - j) * H), scale,
                                              *pat, sparse=True, causal=True)
        assert _norm_err(dk[bi, j].double().cpu().numpy()[None], rk[j][None]) <= 2e-2
        assert _norm_err(dv[bi, j].double().cpu().numpy()[None], rv[j][None]) <= 2e-2
