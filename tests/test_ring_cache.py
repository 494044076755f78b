"""Bounded SSA KV cache.

CPU: the ring layout (sink rows [0, s*b), block kb >= s at s*b + ((kb - s) mod l)*b) against an independent
model of SPEC's SsaKvCache (sink store + list of local blocks, a block expires when qb - kb >= l and kb >= s):
after any sequence of appends the slots that hold live rows are exactly {j : allowed(t, j)} for the next query
t (the oracle's mask), and no two live rows share a slot.
GPU: ssa_ring_append contents against that model (bitwise rows), ssa_decode_ring bitwise equal to the
contiguous-cache decode, and token-by-token streaming (append 1 row, decode) against the prefill rows.
"""
import numpy as np
import pytest
import torch

import oracle
from inputs import TID_K, TID_Q, Spec, gen_rows_f32
from inputs.device import empty_filled

D_QK = 576


def ring_slot(j, s, l, b):
    kb = j // b
    return j if kb < s else s * b + ((kb - s) % l) * b + (j - kb * b)


class SpecSsaCache:
    """SPEC.md:369-374 / 397: sink store (first s blocks) + the most recent local blocks; a local block expires
    when a new block opens and qb - kb >= l (kb >= s). Holds absolute positions."""

    def __init__(self, s, l, b):
        self.s, self.l, self.b = s, l, b
        self.sink, self.local, self.t = [], {}, 0

    def append(self, j):
        assert j == self.t
        kb = j // self.b
        if kb < self.s:
            self.sink.append(j)
        else:
            self.local.setdefault(kb, []).append(j)
            for old in [k for k in self.local if kb - k >= self.l]:  # block-boundary eviction
                del self.local[old]
        self.t += 1

    def retained(self):
        return sorted(self.sink + [j for v in self.local.values() for j in v])


@pytest.mark.parametrize("pat", [(1, 2, 128), (1, 7, 128), (2, 3, 128), (1, 3, 256), (0, 4, 128)])
def test_ring_layout_matches_spec_cache(pat):
    s, l, b = pat
    cache = SpecSsaCache(s, l, b)
    for t in range(0, 12 * b + 37):
        if t > 0:
            # retained set == {j : allowed(t_query = t - 1 ... )}: the cache serves the query at the last position
            ret = cache.retained()
            allowed = oracle.allowed_keys(t - 1, t, s, l, b).tolist()
            assert ret == allowed, (t, ret[:5], allowed[:5])
            slots = [ring_slot(j, s, l, b) for j in ret]
            assert len(set(slots)) == len(slots) and max(slots) < (s + l) * b
        cache.append(t)


pytestmark_gpu = pytest.mark.gpu


def _mk(seed, B, n, H=64):
    qs = Spec(seed=seed, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK)
    ks = Spec(seed=seed, tensor_id=TID_K, batch=B, n=n, heads=1, d=D_QK)
    return qs, ks


@pytest.mark.gpu
@pytest.mark.parametrize("pat", [(1, 2, 128), (2, 3, 128), (1, 3, 256)])
def test_append_contents_match_spec_model(pat):
    from paper_2512_23966_b200 import loza
    s, l, b = pat
    B, n = 3, 9 * b + 77
    _, ks = _mk(31, B, n)
    kv = empty_filled(ks)  # [B, n, 576] source rows
    R = (s + l) * b
    cache = torch.zeros((B, R, D_QK), dtype=torch.bfloat16, device="cuda")
    # different chunkings per sequence, all ending at n: prompt chunk, then single tokens, then a chunk
    cuts = [[0, 300, 301, 302, n], [0, 1, 2, b, b + 1, n], [0, n]]
    models = [SpecSsaCache(s, l, b) for _ in range(B)]
    steps = max(len(c) for c in cuts) - 1
    for k in range(steps):
        # one append call per step: sequences that are done get m = 0 rows via a 0-length chunk (skip them)
        for bi in range(B):
            if k + 1 >= len(cuts[bi]):
                continue
            p0, p1 = cuts[bi][k], cuts[bi][k + 1]
            pos0 = torch.tensor([p0], dtype=torch.int32, device="cuda")
            loza.ssa_ring_append(cache[bi:bi + 1], kv[bi:bi + 1, p0:p1], pos0, pattern=pat)
            for j in range(p0, p1):
                models[bi].append(j)
    torch.cuda.synchronize()
    for bi in range(B):
        for j in models[bi].retained():
            assert torch.equal(cache[bi, ring_slot(j, s, l, b)], kv[bi, j]), (bi, j)


@pytest.mark.gpu
@pytest.mark.parametrize("pat", [(1, 7, 128), (2, 3, 128), (1, 3, 256)])
def test_ring_decode_bitwise_equals_contiguous(pat):
    from paper_2512_23966_b200 import loza
    s, l, b = pat
    lens = [1, 100, (s + l) * b, (s + l) * b + 1, 5 * b + 17, 40000, 65536 + 3, 7 * b]
    B = len(lens)
    T = max(lens)
    qs, ks = _mk(32, B, T)
    q, kv = empty_filled(qs), empty_filled(ks)
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    ref = loza.ssa_decode(q, kv, seq, pattern=pat)
    cache = torch.zeros((B, (s + l) * b, D_QK), dtype=torch.bfloat16, device="cuda")
    for bi, L in enumerate(lens):  # a whole prompt per sequence (m = L, pos0 = 0)
        loza.ssa_ring_append(cache[bi:bi + 1], kv[bi:bi + 1, :L], torch.zeros(1, dtype=torch.int32, device="cuda"),
                             pattern=pat)
    got = loza.ssa_decode_ring(q, cache, seq, pattern=pat)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


@pytest.mark.gpu
def test_streaming_decode_matches_prefill_rows():
    """append a prompt, then one token at a time; each decode equals the oracle row of the whole sequence."""
    from paper_2512_23966_b200 import loza
    pat = (1, 2, 128)
    s, l, b = pat
    B, n, p0 = 2, 700, 384
    ks = Spec(seed=33, tensor_id=TID_K, batch=B, n=n, heads=1, d=D_QK)
    qs = Spec(seed=33, tensor_id=TID_Q, batch=B, n=n, heads=64, d=D_QK)
    kv, q = empty_filled(ks), empty_filled(qs)
    cache = torch.zeros((B, (s + l) * b, D_QK), dtype=torch.bfloat16, device="cuda")
    loza.ssa_ring_append(cache, kv[:, :p0], torch.zeros(B, dtype=torch.int32, device="cuda"), pattern=pat)
    scale = loza.default_scale(D_QK)
    for t in [p0, p0 + 1, 511, 512, 513, 640, n - 1]:
        while int(t) > p0:  # append rows up to t - 1 one at a time
            loza.ssa_ring_append(cache, kv[:, p0:p0 + 1], torch.full((B,), p0, dtype=torch.int32, device="cuda"),
                                 pattern=pat)
            p0 += 1
        loza.ssa_ring_append(cache, kv[:, t:t + 1], torch.full((B,), t, dtype=torch.int32, device="cuda"),
                             pattern=pat)
        p0 = t + 1
        seq = torch.full((B,), t + 1, dtype=torch.int32, device="cuda")
        o = loza.ssa_decode_ring(q[:, t:t + 1], cache, seq, pattern=pat)
        torch.cuda.synchronize()
        for bi in range(B):
            kf = gen_rows_f32(ks, bi * n, t + 1)
            qr = gen_rows_f32(qs, (bi * n + t) * 64, 64)
            ref, _ = oracle.attention_rows(qr, np.full(64, t), kf, kf[:, :512], scale, *pat)
            assert np.abs(o[bi, 0].double().cpu().numpy() - ref).max() <= 2e-2, (t, bi)
