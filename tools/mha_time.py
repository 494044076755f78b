"""Time ssa_prefill_mha (f4) at the bench shape: B1, 32K tokens, H 64, (1,7,128); algorithmic flops per
(token, head) = 2 * (192 + 128) * |allowed keys|."""
import sys
import numpy as np
import torch
from inputs import TID_K, TID_Q, TID_V, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
H = int(sys.argv[2]) if len(sys.argv) > 2 else 64
pat = (1, 7, 128)
q, k, v = (empty_filled(Spec(seed=7, tensor_id=t, batch=1, n=n, heads=H, d=d), four_d=True)
           for t, d in ((TID_Q, 192), (TID_K, 192), (TID_V, 128)))
o = torch.empty((1, n, H, 128), dtype=torch.bfloat16, device="cuda")
s, l, b = pat
# exact count via the oracle-free closed form: sink blocks + local blocks (causal)
cnt = 0
for i in range(n):
    B_ = i // b
    sink = [j for j in range(min(s, B_ + 1))]
    loc = [j for j in range(max(s, B_ - l + 1), B_ + 1)]
    cnt += sum(min(b, i + 1 - j * b) for j in set(sink) | set(loc))
flops = 2.0 * (192 + 128) * cnt * H
for _ in range(3):
    loza.ssa_prefill_mha(q, k, v, pat, out=o)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(10):
    ev[0].record(); loza.ssa_prefill_mha(q, k, v, pat, out=o); ev[1].record(); torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ms = float(np.median(ts))
print(f"mha n={n} H={H}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s  {n / ms * 1e3 / 1e6:.2f} Mtok/s")
full = loza.ssa_prefill_mha(q, k, v, sparse=False)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    ev[0].record(); loza.ssa_prefill_mha(q, k, v, sparse=False, out=o); ev[1].record(); torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ffl = 2.0 * (192 + 128) * (n * (n + 1) / 2) * H
print(f"mha full n={n}: {np.median(ts):.3f} ms  {ffl / np.median(ts) / 1e9:.1f} TFLOP/s")
