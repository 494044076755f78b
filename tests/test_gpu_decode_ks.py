"""Head-sharded decode (SURVEY.md §8 a7 and e) and the key-split pair decode kernel (attn_tc_decode_ks.cu).

- H < 64 (north star: decode "shards by batch and heads"): every GPU of a head-sharded decode runs
  ssa_decode with its H/R heads over the same latent window (the pair-cooperative kernel with zero-padded
  heads by default; the key-split kernel through test knob decode = 2). Against the fp64 oracle on ragged
  seq_lens, both output dtypes, LSE, four patterns, and the bounded ring cache.
- H == 64 through the same kernel (test knob decode = 2): the whole decode + ring parity suites re-run in a
  subprocess (the library never reads the environment; tests/conftest.py applies LOZA_TEST_DECODE_KERNEL).
- The decode workspace's status word: a seq_len outside [1, n_kv] is reported (LOZA_ERR_SHAPE), the row is
  computed at the clamped length.
"""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from inputs import TID_K, TID_Q, Spec, gen_rows_f32, gen_rows_f32_at
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu

D_QK, D_V = 576, 512
SCALE = loza.default_scale(576)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle(qs, ks, bi, L, pattern, H):
    s, l, b = pattern
    keys = oracle.allowed_keys(L - 1, L, s, l, b)
    kf = gen_rows_f32_at(ks, bi * ks.n + keys)
    qr = gen_rows_f32(qs, bi * H, H)
    return oracle.attend(qr, kf, kf[:, :D_V], SCALE)


@pytest.mark.parametrize("H", [1, 8, 16, 32, 48, 63])
@pytest.mark.parametrize("pattern", [(1, 7, 128), (2, 3, 256), (0, 3, 128)])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_decode_head_sharded_vs_oracle(H, pattern, out_dtype):
    seq = [1, 64, 65, 128, 1000, 1024, 1025, 2048, 4000]
    B, T = len(seq), 4096
    qs = Spec(seed=91 + H, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    ks = Spec(seed=91 + H, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK, kind="kv_marker", block=pattern[2],
              marker_mod=D_V, amp=0.5)
    q, cache = empty_filled(qs), empty_filled(ks)
    sl = torch.tensor(seq, dtype=torch.int32, device="cuda")
    lse = torch.full((B, H, 1), float("nan"), device="cuda")
    o = loza.ssa_decode(q, cache, sl, pattern=pattern, scale=SCALE, lse=lse, out_dtype=out_dtype)
    torch.cuda.synchronize()
    for bi, L in enumerate(seq):
        ref, rl = _oracle(qs, ks, bi, L, pattern, H)
        got = o[bi, 0].double().cpu().numpy()
        assert np.abs(got - ref).max() <= 2e-2, (bi, L)
        assert np.abs(lse[bi, :, 0].double().cpu().numpy() - rl).max() <= 1e-3 * max(1.0, np.abs(rl).max()), bi


@pytest.mark.parametrize("H", [16, 32])
def test_decode_ring_head_sharded_equals_contiguous(H):
    """The bounded ring cache at H < 64 gives the contiguous-cache decode's bits."""
    pattern, B, T = (1, 7, 128), 6, 3000
    seq = [1, 200, 1024, 1500, 2047, 3000]
    s, l, b = pattern
    qs = Spec(seed=95, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    ks = Spec(seed=95, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    q, cache = empty_filled(qs), empty_filled(ks)
    ring = torch.zeros((B, (s + l) * b, D_QK), dtype=torch.bfloat16, device="cuda")
    for bi, L in enumerate(seq):
        loza.ssa_ring_append(ring[bi:bi + 1], cache[bi:bi + 1, :L], torch.zeros(1, dtype=torch.int32, device="cuda"),
                             pattern=pattern)
    sl = torch.tensor(seq, dtype=torch.int32, device="cuda")
    o_ring = loza.ssa_decode_ring(q, ring, sl, pattern=pattern, scale=SCALE)
    o_cont = loza.ssa_decode(q, cache, sl, pattern=pattern, scale=SCALE)
    torch.cuda.synchronize()
    assert torch.equal(o_ring, o_cont)


def test_decode_status_word_reports_clamped_seq_len():
    H, B, T, pattern = 64, 4, 2048, (1, 7, 128)
    qs = Spec(seed=97, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    ks = Spec(seed=97, tensor_id=TID_K, batch=B, n=T, heads=1, d=D_QK)
    q, cache = empty_filled(qs), empty_filled(ks)
    a = loza.make_args(q, cache, cache[..., :D_V], torch.empty((B, 1, H, D_V), dtype=torch.bfloat16, device="cuda"),
                       scale=SCALE)
    need = loza.lib().loza_workspace_size(loza.LOZA_WS_DECODE, a, loza.Pattern(*pattern), 1)
    assert need >= 4
    ws = torch.full((need,), 0xAB, dtype=torch.uint8, device="cuda")
    assert loza.lib().loza_workspace_init(loza.LOZA_WS_DECODE, a, loza.Pattern(*pattern), 1,
                                          ws.data_ptr(), need, None) == 0
    ok = torch.tensor([100, 2048, 1, 500], dtype=torch.int32, device="cuda")
    loza.ssa_decode(q, cache, ok, pattern=pattern, scale=SCALE, ws=ws)
    assert loza.decode_status(ws) == 0
    bad = torch.tensor([100, 5000, 1, 0], dtype=torch.int32, device="cuda")  # 5000 > n_kv, 0 < 1
    o = loza.ssa_decode(q, cache, bad, pattern=pattern, scale=SCALE, ws=ws, out_dtype=torch.float32)
    assert loza.decode_status(ws) == 2  # LOZA_ERR_SHAPE
    ref, _ = _oracle(qs, ks, 1, T, pattern, H)  # computed at the clamped length
    assert np.abs(o[1, 0].double().cpu().numpy() - ref).max() <= 2e-2
    loza.decode_status_reset(ws)
    loza.ssa_decode(q, cache, ok, pattern=pattern, scale=SCALE, ws=ws)
    assert loza.decode_status(ws) == 0


def test_key_split_kernel_through_the_h64_parity_suites():
    env = dict(os.environ, LOZA_TEST_DECODE_KERNEL="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_tc_decode.py"),
                        os.path.join(ROOT, "tests", "test_ring_cache.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_key_split_kernel_head_sharded():
    """The key-split kernel (test knob decode = 2) through the H < 64 parity cases above."""
    env = dict(os.environ, LOZA_TEST_DECODE_KERNEL="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "head_sharded_vs_oracle or ring_head_sharded",
                        os.path.join(ROOT, "tests", "test_gpu_decode_ks.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
