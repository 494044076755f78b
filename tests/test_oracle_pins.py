"""Pins for the fp64 CPU oracle (oracle/), against what the paper and mathematics fix.

None of these re-types the oracle's formulas. Each pin is one of: a value the
paper / SPEC prints (tests/golden/, cited), a closed form, a library routine
(torch SDPA in fp64), brute force on tiny inputs by an independent route, or an
invariant. A plausible mistake anywhere in the oracle (wrong sign / index in the
mask, own block not counted as local, dropped scale, transposed operand, wrong
blend coefficient) fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- mask / selection
def test_mask_hand_example_spec124():
    g = _gold("spec124_mask_example.json")
    for tok, want in g["attends"].items():
        got = oracle.allowed_keys(int(tok), g["n"], g["s"], g["l"], g["b"])
        assert got.tolist() == want, (tok, got)


def test_window_is_1024_paper97():
    g = _gold("paper97_pattern.json")
    s, l, b = g["s"], g["l"], g["b"]
    assert (s + l) * b == g["window_tokens"]
    t = g["decode_context"]
    # decode: the current token sits at p = t - 1 (reading R8)
    keys = oracle.allowed_keys(t - 1, t, s, l, b)
    assert len(keys) == g["decode_rows_read"]
    # the window is the sink block plus the last l blocks (own block included, reading R2)
    assert keys[:b].tolist() == list(range(b))
    assert keys[b:].tolist() == list(range(t - l * b, t))


def test_dense_causal_degeneracy_spec125_126():
    g = _gold("spec125_dense_cases.json")
    for c in g["cases"]:
        for p in range(c["n"]):
            assert oracle.allowed_keys(p, c["n"], c["s"], c["l"], c["b"]).tolist() == list(range(p + 1))
    rng = np.random.default_rng(0)
    for _ in range(40):
        s, l, b = int(rng.integers(0, 4)), int(rng.integers(1, 5)), int(rng.integers(1, 9))
        n = int(rng.integers(1, (s + l) * b + 1))
        for p in range(n):
            m = oracle.mask_row(p, n, s, l, b)
            assert m.tolist() == [1] * (p + 1) + [0] * (n - p - 1)


def test_full_mask_is_causal_and_bidirectional():
    for p in range(7):
        assert oracle.mask_row(p, 7, 0, 1, 1, sparse=False).tolist() == [1] * (p + 1) + [0] * (6 - p)
        assert oracle.mask_row(p, 7, 0, 1, 1, sparse=False, causal=False).tolist() == [1] * 7


def test_selection_closed_form_and_counts():
    """|sel(qb)| = min(qb+1, s+l) and sel(qb) = {0..s-1} U {qb-l+1..qb} (for full blocks), by exhaustive
    brute force over n <= 512 x random patterns."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        s, l, b = int(rng.integers(0, 4)), int(rng.integers(1, 6)), int(rng.integers(1, 40))
        n = int(rng.integers(1, 513))
        idx, cnt = oracle.select_blocks(n, 0, n, s, l, b)
        for qb in range(len(cnt)):
            want = sorted(set(range(min(s, qb + 1))) | set(range(max(0, qb - l + 1), qb + 1)))
            assert cnt[qb] == len(want) == min(qb + 1, len(want))
            assert idx[qb, :cnt[qb]].tolist() == want
            assert (idx[qb, cnt[qb]:] == -1).all()
            assert cnt[qb] == min(qb + 1, s + l) or s > qb  # sinks overlap the local run near the start


def test_selection_with_q_start_offsets():
    s, l, b, n = 1, 3, 16, 400
    full_idx, full_cnt = oracle.select_blocks(n, 0, n, s, l, b)
    qs = 96
    idx, cnt = oracle.select_blocks(n - qs, qs, n, s, l, b)
    assert (idx == full_idx[qs // b:]).all() and (cnt == full_cnt[qs // b:]).all()


def _pairs_closed_form(n, s, l, b):
    # SURVEY.md §8 (pair counts): n = N*b, N-1 >= W = s+l-1, s = 1
    N, W = n // b, s + l - 1
    return b * b * (W * (W + 1) // 2 + (N - 1 - W) * W) + N * b * (b + 1) // 2


def test_pair_counts_brute_force():
    # tiny config (1,2,64), n 1024 -> 152,064 pairs; a few other shapes by the closed form
    for (n, s, l, b) in [(1024, 1, 2, 64), (2048, 1, 7, 128), (640, 1, 3, 32)]:
        tot = sum(len(oracle.allowed_keys(p, n, s, l, b)) for p in range(n))
        assert tot == _pairs_closed_form(n, s, l, b)
    assert _pairs_closed_form(1024, 1, 2, 64) == 152064


# ----------------------------------------------------------------------------- attention
def _sdpa64(q, k, v, scale, mask):
    """torch SDPA in fp64 (library routine). q [R,d], k [n,d], v [n,dv], mask [R,n] bool."""
    qt = torch.from_numpy(q.astype(np.float64))[None, None]
    kt = torch.from_numpy(k.astype(np.float64))[None, None]
    vt = torch.from_numpy(v.astype(np.float64))[None, None]
    m = torch.from_numpy(mask)[None, None]
    return torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=m, scale=scale)[0, 0].numpy()


def test_full_attention_matches_sdpa_is_causal():
    rng = np.random.default_rng(2)
    n, d, dv = 37, 16, 12
    q = rng.standard_normal((n, d)).astype(np.float32)
    k = rng.standard_normal((n, d)).astype(np.float32)
    v = rng.standard_normal((n, dv)).astype(np.float32)
    scale = 0.3
    o, lse = oracle.attention_rows(q, np.arange(n), k, v, scale, sparse=False)
    qt, kt, vt = (torch.from_numpy(x.astype(np.float64))[None, None] for x in (q, k, v))
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, scale=scale)[0, 0].numpy()
    assert np.abs(o - ref).max() < 1e-12
    # LSE against torch.logsumexp of the causal logits
    z = torch.from_numpy(q.astype(np.float64)) @ torch.from_numpy(k.astype(np.float64)).T * scale
    z = z.masked_fill(torch.ones(n, n, dtype=torch.bool).triu(1), float("-inf"))
    assert np.abs(lse - torch.logsumexp(z, dim=1).numpy()).max() < 1e-12


def test_ssa_matches_sdpa_with_explicit_mask():
    rng = np.random.default_rng(3)
    for (n, s, l, b) in [(50, 1, 2, 4), (64, 2, 1, 8), (33, 0, 3, 5)]:
        d, dv = 8, 6
        q = rng.standard_normal((n, d)).astype(np.float32)
        k = rng.standard_normal((n, d)).astype(np.float32)
        v = rng.standard_normal((n, dv)).astype(np.float32)
        mask = np.stack([oracle.mask_row(p, n, s, l, b).astype(bool) for p in range(n)])
        o, _ = oracle.attention_rows(q, np.arange(n), k, v, 0.5, s, l, b)
        assert np.abs(o - _sdpa64(q, k, v, 0.5, mask)).max() < 1e-12


def test_ssa_equals_full_when_window_covers():
    rng = np.random.default_rng(4)
    for _ in range(100):  # SPEC.md:165 (100 random trials)
        s, l, b = int(rng.integers(0, 3)), int(rng.integers(1, 4)), int(rng.integers(1, 6))
        n = int(rng.integers(1, (s + l) * b + 1))
        q, k = rng.standard_normal((2, n, 4)).astype(np.float32)
        v = rng.standard_normal((n, 3)).astype(np.float32)
        o1, _ = oracle.attention_rows(q, np.arange(n), k, v, 0.7, s, l, b)
        o2, _ = oracle.attention_rows(q, np.arange(n), k, v, 0.7, sparse=False)
        assert np.abs(o1 - o2).max() < 1e-12


def test_closed_forms():
    rng = np.random.default_rng(5)
    n, d = 9, 5
    q, k = rng.standard_normal((2, n, d)).astype(np.float32)
    v = rng.standard_normal((n, 4)).astype(np.float32)
    # (s=0, l=1, b=1): each token attends only itself => O = V
    o, lse = oracle.attention_rows(q, np.arange(n), k, v, 1.0, 0, 1, 1)
    assert np.array_equal(o, v.astype(np.float64))
    # n = 1 => O = V
    o1, _ = oracle.attention_rows(q[:1], [0], k[:1], v[:1], 1.0, sparse=False)
    assert np.array_equal(o1[0], v[0].astype(np.float64))
    # Q = 0, n = 2 => row 1 = (V0 + V1)/2 and LSE = ln 2
    o2, l2 = oracle.attention_rows(np.zeros((1, d), np.float32), [1], k[:2], v[:2], 1.0, sparse=False)
    assert np.abs(o2[0] - (v[0].astype(np.float64) + v[1]) / 2).max() < 1e-15
    assert abs(l2[0] - math.log(2)) < 1e-15
    # two-key logistic closed form (checks the scale and that K is transposed): q=1, k0=0, k1=1
    q1 = np.array([[1.0, 0.0]], np.float32)
    kk = np.array([[0.0, 0.0], [1.0, 0.0]], np.float32)
    vv = np.array([[0.0], [1.0]], np.float32)
    for scale in (1.0, 0.25, 3.0):
        o3, l3 = oracle.attention_rows(q1, [1], kk, vv, scale, sparse=False)
        assert abs(o3[0, 0] - 1.0 / (1.0 + math.exp(-scale))) < 1e-15
        assert abs(l3[0] - math.log(1.0 + math.exp(scale))) < 1e-14


def test_uniform_and_constant_cases_ssa():
    rng = np.random.default_rng(6)
    n, s, l, b = 40, 1, 2, 4
    k = rng.standard_normal((n, 6)).astype(np.float32)
    v = rng.standard_normal((n, 3)).astype(np.float32)
    o, lse = oracle.attention_rows(np.zeros((n, 6), np.float32), np.arange(n), k, v, 1.0, s, l, b)
    for p in range(n):
        # allowed set counted by hand: sink block [0,4) plus blocks qb-1, qb up to p
        qb = p // b
        allowed = sorted(set(range(min(b, p + 1))) | set(range(max(0, (qb - l + 1) * b), p + 1)))
        assert np.abs(o[p] - v[allowed].astype(np.float64).mean(0)).max() < 1e-14
        assert abs(lse[p] - math.log(len(allowed))) < 1e-14
    # V = c => O = c (rows of the softmax sum to one)
    c = np.full((n, 3), 0.375, np.float32)
    oc, _ = oracle.attention_rows(rng.standard_normal((n, 6)).astype(np.float32), np.arange(n), k, c, 0.9, s, l, b)
    assert np.abs(oc - 0.375).max() < 1e-15


def test_perturbation_invariance_spec167_168():
    rng = np.random.default_rng(7)
    n, s, l, b = 6, 1, 1, 2
    q, k = rng.standard_normal((2, n, 3)).astype(np.float32)
    v = rng.standard_normal((n, 2)).astype(np.float32)
    o, _ = oracle.attention_rows(q, np.arange(n), k, v, 1.0, s, l, b)
    k2, v2 = k.copy(), v.copy()
    k2[2:4] += 5.0
    v2[2:4] -= 7.0  # rows 2-3 are outside token 4's and 5's window
    o2, _ = oracle.attention_rows(q, np.arange(n), k2, v2, 1.0, s, l, b)
    assert np.array_equal(o[4:], o2[4:])
    assert not np.allclose(o[2:4], o2[2:4])
    # causality: perturbing j > i never changes row i
    k3 = k.copy()
    k3[5] += 3.0
    o3, _ = oracle.attention_rows(q, np.arange(n), k3, v, 1.0, s, l, b)
    assert np.array_equal(o[:5], o3[:5])


def test_decode_is_last_row_of_prefill_spec398():
    rng = np.random.default_rng(8)
    n, s, l, b = 70, 1, 2, 8
    q, k = rng.standard_normal((2, n, 5)).astype(np.float32)
    v = rng.standard_normal((n, 4)).astype(np.float32)
    o, lse = oracle.attention_rows(q, np.arange(n), k, v, 0.6, s, l, b)
    for t in (1, 9, 17, 64, 70):
        od, ld = oracle.attention_rows(q[t - 1:t], [t - 1], k[:t], v[:t], 0.6, s, l, b)
        assert np.abs(od[0] - o[t - 1]).max() < 1e-14 and abs(ld[0] - lse[t - 1]) < 1e-14


def test_attend_gathered_equals_masked_rows():
    rng = np.random.default_rng(9)
    n, s, l, b = 300, 1, 3, 16
    q, k = rng.standard_normal((2, n, 7)).astype(np.float32)
    v = rng.standard_normal((n, 5)).astype(np.float32)
    for p in (0, 15, 16, 100, 299):
        keys = oracle.allowed_keys(p, n, s, l, b)
        og, lg = oracle.attend(q[p:p + 1], k[keys], v[keys], 0.4)
        om, lm = oracle.attention_rows(q[p:p + 1], [p], k, v, 0.4, s, l, b)
        assert np.abs(og - om).max() < 1e-14 and abs(lg[0] - lm[0]) < 1e-13


def test_attention_batched_wrapper_layout():
    rng = np.random.default_rng(10)
    B, n, H, d, dv = 2, 20, 3, 6, 4
    q = rng.standard_normal((B, n, H, d)).astype(np.float32)
    k = rng.standard_normal((B, n, d)).astype(np.float32)
    v = rng.standard_normal((B, n, dv)).astype(np.float32)
    o, lse = oracle.attention(q, k, v, 0.5, (1, 2, 4))
    for bi, t, h in itertools.product(range(B), (0, 7, 19), range(H)):
        mask = oracle.mask_row(t, n, 1, 2, 4).astype(bool)[None]
        ref = _sdpa64(q[bi, t, h][None], k[bi], v[bi], 0.5, mask)[0]
        assert np.abs(o[bi, t, h] - ref).max() < 1e-12
        assert lse.shape == (B, H, n)


# ----------------------------------------------------------------------------- blend (Eq. 3)
def test_blend_endpoints_and_hand_values():
    rng = np.random.default_rng(11)
    o = rng.standard_normal(1000).astype(np.float32)
    op = rng.standard_normal(1000).astype(np.float32)
    d = rng.standard_normal(1000).astype(np.float32)
    h1, _ = oracle.blend(o, op, 1.0)
    h0, _ = oracle.blend(o, op, 0.0)
    assert np.array_equal(h1, o.astype(np.float64)) and np.array_equal(h0, op.astype(np.float64))
    hh, _ = oracle.blend(o, o, 0.37)  # O == O' => O^ == O for any alpha
    assert np.abs(hh - o).max() < 1e-15
    _, da = oracle.blend(np.array([1, 2], np.float32), np.array([0, 1], np.float32), 0.5,
                         np.array([3, 4], np.float32))
    assert da == 7.0  # 3*(1-0) + 4*(2-1), by hand
    h, _ = oracle.blend(np.array([2.0], np.float32), np.array([6.0], np.float32), 0.25)
    assert h[0] == 5.0  # 0.25*2 + 0.75*6, by hand


def test_blend_gradient_finite_difference_spec170():
    rng = np.random.default_rng(12)
    o, op, d = rng.standard_normal((3, 4096)).astype(np.float32)
    for a in (0.1, 0.5, 0.9):
        _, da = oracle.blend(o, op, a, d)
        eps = 1e-3
        lp = float(np.dot(d.astype(np.float64), oracle.blend(o, op, a + eps)[0]))
        lm = float(np.dot(d.astype(np.float64), oracle.blend(o, op, a - eps)[0]))
        assert abs((lp - lm) / (2 * eps) - da) <= 1e-9 * np.abs(d.astype(np.float64) * (o - op)).sum()


# ---------------------------------------------------------------- attention backward
def _loss(q, pos, k, v, do, scale, pat, sparse=True, causal=True):
    o, _ = oracle.attention_rows(q, pos, k, v, scale, *pat, sparse=sparse, causal=causal)
    return float((o * do.astype(np.float64)).sum())


@pytest.mark.parametrize("sparse", [True, False])
def test_backward_finite_differences(sparse):
    """Central differences of L = sum dO . O(Q, K, V) through the FORWARD oracle (independent of the backward
    formulas) on random entries of q, k and v; h = 2^-10 is exact in fp32 for |x| < 2^13."""
    rng = np.random.default_rng(7)
    pat = (1, 2, 4)
    R, n_kv, dqk, dv = 9, 20, 6, 5
    pos = np.array([0, 3, 4, 7, 8, 12, 15, 18, 19], dtype=np.int64)
    q = rng.standard_normal((R, dqk)).astype(np.float32)
    k = rng.standard_normal((n_kv, dqk)).astype(np.float32)
    v = rng.standard_normal((n_kv, dv)).astype(np.float32)
    do = rng.standard_normal((R, dv)).astype(np.float32)
    scale = 0.7
    dq, dk, dvv = oracle.attention_backward(q, pos, k, v, do, scale, *pat, sparse=sparse)
    h = 2.0 ** -10
    for arr, grad in ((q, dq), (k, dk), (v, dvv)):
        for idx in [tuple(rng.integers(0, d) for d in arr.shape) for _ in range(12)]:
            xp, xm = arr.copy(), arr.copy()
            xp[idx] += h
            xm[idx] -= h
            if arr is q:
                lp, lm = _loss(xp, pos, k, v, do, scale, pat, sparse), _loss(xm, pos, k, v, do, scale, pat, sparse)
            elif arr is k:
                lp, lm = _loss(q, pos, xp, v, do, scale, pat, sparse), _loss(q, pos, xm, v, do, scale, pat, sparse)
            else:
                lp, lm = _loss(q, pos, k, xp, do, scale, pat, sparse), _loss(q, pos, k, xm, do, scale, pat, sparse)
            fd = (lp - lm) / (2 * h)
            assert abs(fd - grad[idx]) <= 1e-5 * max(1.0, abs(grad[idx])), (idx, fd, grad[idx])


def test_backward_single_key_and_constant_v():
    """One allowed key: P = 1, so dq = dk = 0 and dv = sum of dO over the rows. V rows all equal: O = v for any
    P, so dq = dk = 0 and dv_j = sum_r P_rj dO_r (sums to sum dO over keys)."""
    rng = np.random.default_rng(8)
    R, dqk, dv = 5, 4, 3
    q = rng.standard_normal((R, dqk)).astype(np.float32)
    do = rng.standard_normal((R, dv)).astype(np.float32)
    k1 = rng.standard_normal((1, dqk)).astype(np.float32)
    v1 = rng.standard_normal((1, dv)).astype(np.float32)
    dq, dk, dvv = oracle.attention_backward(q, np.zeros(R, dtype=np.int64), k1, v1, do, 0.5, 0, 1, 1, sparse=False)
    assert np.abs(dq).max() < 1e-14 and np.abs(dk).max() < 1e-14
    assert np.allclose(dvv[0], do.astype(np.float64).sum(0), rtol=0, atol=1e-12)
    n_kv = 6
    kc = rng.standard_normal((n_kv, dqk)).astype(np.float32)
    vc = np.tile(rng.standard_normal((1, dv)).astype(np.float32), (n_kv, 1))
    pos = np.full(R, n_kv - 1, dtype=np.int64)
    dq, dk, dvv = oracle.attention_backward(q, pos, kc, vc, do, 0.5, 0, 1, 1, sparse=False)
    assert np.abs(dq).max() < 1e-12 and np.abs(dk).max() < 1e-12
    assert np.allclose(dvv.sum(0), do.astype(np.float64).sum(0), rtol=0, atol=1e-12)


@pytest.mark.parametrize("sparse", [True, False])
def test_backward_gradient_identities(sparse):
    """Identities of the softmax gradient that hold at any size (also checked on the GPU at 8K,
    tests/test_gpu_fullsize.py): sum_j P_rj = 1 gives sum_j dV_j = sum_r dO_r; sum_j dS_rj = D_r - D_r = 0
    gives sum_j dK_j = 0. A dropped sink or window block, or a wrong D, breaks them."""
    rng = np.random.default_rng(9)
    pat = (1, 2, 4)
    n_kv, dqk, dv = 40, 7, 5
    pos = np.repeat(np.arange(n_kv), 2)  # two heads per position
    q = rng.standard_normal((len(pos), dqk)).astype(np.float32)
    k = rng.standard_normal((n_kv, dqk)).astype(np.float32)
    v = rng.standard_normal((n_kv, dv)).astype(np.float32)
    do = rng.standard_normal((len(pos), dv)).astype(np.float32)
    dq, dk, dvv = oracle.attention_backward(q, pos, k, v, do, 0.6, *pat, sparse=sparse)
    assert np.abs(dvv.sum(0) - do.astype(np.float64).sum(0)).max() <= 1e-12 * max(1.0, np.abs(dvv).sum())
    assert np.abs(dk.sum(0)).max() <= 1e-12 * max(1.0, np.abs(dk).sum())
