"""The 1M-token SSA prefill (BASELINE.json configs[4]; "up to 1 million tokens", PAPER.md:97 the
(1,7,128) pattern at 1M) on ONE GPU, in the launch configuration bench.py times: B1, n = 1,048,576, H64, MLA
576/512, bf16 in / bf16 out, LSE on. Q is 77.3 GB, O 68.7 GB, so the unit decode, TMA coordinates and output /
LSE offsets run at 2^26 rows.

Sampled (token, all 64 heads) rows against the fp64 oracle: the oracle derives the row's allowed keys from its
own explicit mask (oracle.allowed_keys), the rows are regenerated from the counter-based generator,
and oracle.attend computes softmax(scale q k^T) v over exactly those keys. Tolerance as everywhere for bf16
(R12): max-abs <= 2e-2, normwise guard <= 1e-2, LSE within 1e-3 relative.
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_K, TID_Q, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

H, D_QK, D_V = 64, 576, 512
PAT = (1, 7, 128)
N = 1 << 20


def _need_bytes():
    return N * H * (D_QK + D_V) * 2 + N * D_QK * 2 + H * N * 4


def _n_allowed(t):
    """Closed-form window size at position t: own block up to t, the l-1 previous blocks, the sink blocks
    not already among them (DESIGN R2, R4, R5)."""
    s, l, b = PAT
    qb = t // b
    lo = max(0, qb - l + 1)
    return t % b + 1 + (qb - lo) * b + min(s, lo) * b


def _oracle_token(qs, ks, t, scale):
    s, l, b = PAT
    keys = oracle.allowed_keys(t, N, s, l, b)
    kf = np.concatenate([gen_rows_f32(ks, int(j), 1) for j in keys])
    qr = gen_rows_f32(qs, t * H, H)
    return oracle.attend(qr, kf, kf[:, :D_V], scale), len(keys)


def test_ssa_prefill_1m_sampled_rows():
    torch.cuda.empty_cache()
    free = torch.cuda.mem_get_info()[0]
    if free < _need_bytes() + (1 << 30):
        pytest.skip(f"needs {_need_bytes() / 1e9:.1f} GB of device memory, {free / 1e9:.1f} GB free")
    qs = Spec(seed=61, tensor_id=TID_Q, batch=1, n=N, heads=H, d=D_QK)
    ks = Spec(seed=61, tensor_id=TID_K, batch=1, n=N, heads=1, d=D_QK)
    q, kv = empty_filled(qs), empty_filled(ks)
    scale = loza.default_scale(D_QK)
    lse = torch.full((1, H, N), float("nan"), device="cuda")
    o = loza.ssa_prefill(q, kv, pattern=PAT, scale=scale, lse=lse)
    torch.cuda.synchronize()
    del q
    rng = np.random.default_rng(61)
    toks = [0, 1, 127, 128, 1023, 1024, 1025, 131071, 131072, 524287, 524288, 524289, 1000000, N - 129, N - 128,
            N - 2, N - 1] + sorted(int(x) for x in rng.integers(0, N, 8))
    for t in toks:
        (ref, rl), nkeys = _oracle_token(qs, ks, t, scale)
        assert nkeys == _n_allowed(t), t
        got = o[0, t].double().cpu().numpy()
        err = np.abs(got - ref).max()
        assert err <= 2e-2, (t, err)
        assert err / np.abs(ref).max() <= 1e-2, (t, err)
        gl = lse[0, :, t].double().cpu().numpy()
        assert np.abs(gl - rl).max() <= 1e-3 * max(1.0, np.abs(rl).max()), t
    # every LSE written (no unit skipped anywhere in the 2^26 rows)
    assert not torch.isnan(lse).any().item()
    del o, lse, kv


def test_ssa_prefill_1m_chunked_equals_whole():
    """The 1M prefill in 8 q_start chunks (the bench's e2e pipeline shape) equals one launch bit for bit: every
    128-row unit is computed the same way whatever the launch it belongs to."""
    n = 1 << 20
    torch.cuda.empty_cache()
    free = torch.cuda.mem_get_info()[0]
    need = n * H * (D_QK + 2 * D_V) * 2 // 8 + n * D_QK * 2 + n * H * D_V * 2
    if free < need + (1 << 30):
        pytest.skip("not enough device memory")
    ks = Spec(seed=62, tensor_id=TID_K, batch=1, n=n, heads=1, d=D_QK)
    kv = empty_filled(ks)
    chunk = n // 8
    scale = loza.default_scale(D_QK)
    for c in (0, 3, 7):
        qs = Spec(seed=62, tensor_id=TID_Q, batch=1, n=n, heads=H, d=D_QK)
        qc = torch.empty((1, chunk, H, D_QK), dtype=torch.bfloat16, device="cuda")
        from inputs.device import fill_
        fill_(qc, qs, row_start=c * chunk * H)
        oc = loza.ssa_prefill(qc, kv[:, :(c + 1) * chunk], pattern=PAT, scale=scale, q_start=c * chunk)
        # the same rows as part of a 2-chunk launch starting one chunk earlier (or later for c = 0)
        c0 = c - 1 if c > 0 else 0
        q2 = torch.empty((1, 2 * chunk, H, D_QK), dtype=torch.bfloat16, device="cuda")
        fill_(q2, qs, row_start=c0 * chunk * H)
        o2 = loza.ssa_prefill(q2, kv[:, :(c0 + 2) * chunk], pattern=PAT, scale=scale, q_start=c0 * chunk)
        torch.cuda.synchronize()
        off = (c - c0) * chunk
        assert torch.equal(oc, o2[:, off:off + chunk]), c
        del qc, q2, oc, o2
