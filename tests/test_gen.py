"""Host-side input generator: determinism, row addressing, statistics, bf16 RNE vs torch."""
import numpy as np
import torch

from inputs import Spec, TID_K, TID_Q, bf16_rne_bits, gen_f32, gen_rows_bits, gen_rows_f32, raw_normal


def test_deterministic_and_row_addressable():
    sp = Spec(seed=3, tensor_id=TID_Q, batch=2, n=40, heads=4, d=24)
    full = gen_f32(sp).reshape(sp.rows, sp.d)
    part = gen_rows_f32(sp, 77, 50)
    assert np.array_equal(full[77:127], part)
    assert np.array_equal(full, gen_f32(sp).reshape(sp.rows, sp.d))
    other = gen_f32(Spec(seed=4, tensor_id=TID_Q, batch=2, n=40, heads=4, d=24))
    assert not np.array_equal(full, other.reshape(sp.rows, sp.d))


def test_unit_statistics():
    z = raw_normal(0, TID_K, np.arange(1 << 20, dtype=np.int64))
    assert abs(float(z.mean())) < 5e-3 and abs(float(z.var()) - 1.0) < 5e-3
    assert float(np.abs(z).max()) <= 3.4642


def test_bf16_rounding_matches_torch():
    z = raw_normal(1, TID_Q, np.arange(1 << 16, dtype=np.int64)) * np.float32(3.7)
    mine = bf16_rne_bits(z)
    ref = torch.from_numpy(z).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(mine, ref)


def test_structures():
    b, dv = 16, 32
    kv = Spec(seed=0, tensor_id=TID_K, batch=1, n=100, heads=1, d=40, kind="kv_marker", block=b,
              marker_mod=dv, amp=0.5)
    plain = Spec(seed=0, tensor_id=TID_K, batch=1, n=100, heads=1, d=40)
    a, p = gen_rows_f32(kv, 0, 100), gen_rows_f32(plain, 0, 100)
    diff = (a != p)
    for j in range(100):
        cols = np.nonzero(diff[j])[0].tolist()
        assert cols in ([(j // b) % dv], [])  # bf16 rounding can hide nothing: +0.5 always shows
    assert diff.sum() >= 95
    sink = Spec(seed=0, tensor_id=TID_K, batch=1, n=100, heads=1, d=40, kind="kv_sink", col=39, sink_rows=16,
                amp=5.0)
    s = gen_rows_f32(sink, 0, 100)
    assert (s[:16, 39] - p[:16, 39] > 4.9).all() and np.array_equal(s[16:], p[16:])
    bits = gen_rows_bits(plain, 0, 3)
    assert bits.dtype == np.uint16
