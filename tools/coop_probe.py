import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
B, ctx = 64, 131072
cache = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=64, d=576))
seq = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
o = torch.empty((B, 1, 64, 512), dtype=torch.bfloat16, device="cuda")
for _ in range(3): loza.ssa_decode(q, cache, seq, out=o)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(10):
    ev[0].record(); loza.ssa_decode(q, cache, seq, out=o); ev[1].record(); torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
print(os.environ.get("LOZA_DECODE_KERNEL", "coop"), "single launch us:", np.round(ts, 1))
ev[0].record()
for _ in range(64): loza.ssa_decode(q, cache, seq, out=o)
ev[1].record(); torch.cuda.synchronize()
print("64 back-to-back (stream, no graph): us/step", ev[0].elapsed_time(ev[1]) * 1e3 / 64)
