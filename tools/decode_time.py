"""Decode step time as bench.py measures it (B64 at 128K, CUDA graph of 64 steps over 4 rotating windows,
L2 flushed before each replay): LOZA_LIB=... python tools/decode_time.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import fill_
from paper_2512_23966_b200 import loza

B, ctx, H, P = 64, 131072, 64, (1, 7, 128)
cache = torch.empty((B, ctx, 576), dtype=torch.bfloat16, device="cuda")
fill_(cache, Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
qd = torch.empty((B, 1, H, 576), dtype=torch.bfloat16, device="cuda")
fill_(qd, Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=H, d=576))
warm = len(sys.argv) > 1 and sys.argv[1] == "warm"  # one window for every step: L2-resident (84 MB < 126 MB)
seqs = [torch.full((B,), ctx - (0 if warm else 2048 * r), dtype=torch.int32, device="cuda") for r in range(4)]
outs = [torch.empty((B, 1, H, 512), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
for r in range(4):
    loza.ssa_decode(qd, cache, seqs[r], pattern=P, out=outs[r])
torch.cuda.synchronize()
R = 64
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
with torch.cuda.stream(cs):
    with torch.cuda.graph(g, stream=cs):
        for i in range(R):
            loza.ssa_decode(qd, cache, seqs[i % 4], pattern=P, out=outs[i % 4])
torch.cuda.synchronize()
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for i in range(12):
    if not warm:
        fl.fill_(i)
    ev[0].record()
    g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(ev[0].elapsed_time(ev[1]) / R * 1e3)
print(f"{os.environ.get('LOZA_LIB', 'default'):32s} {'warm' if warm else 'cold'} decode B64@128K: median {np.median(ts):.2f} us/step  min {min(ts):.2f}")
