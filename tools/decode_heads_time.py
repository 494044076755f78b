"""Head-sharded decode step (B64, H heads of 64, 128K) as bench.py times it: auto kernel vs the key-split kernel
(test knob decode = 2). python tools/decode_heads_time.py [H]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import fill_
from paper_2512_23966_b200 import loza

B, ctx, P = 64, 131072, (1, 7, 128)
Hs = int(sys.argv[1]) if len(sys.argv) > 1 else 32
cache = torch.empty((B, ctx, 576), dtype=torch.bfloat16, device="cuda")
fill_(cache, Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
qd = torch.empty((B, 1, Hs, 576), dtype=torch.bfloat16, device="cuda")
fill_(qd, Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=Hs, d=576))
seqs = [torch.full((B,), ctx - 2048 * r, dtype=torch.int32, device="cuda") for r in range(4)]
outs = [torch.empty((B, 1, Hs, 512), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for knob in (0, 2, 0):
    loza.force_kernel("decode", knob)
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
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for i in range(8):
        fl.fill_(i)
        ev[0].record()
        g.replay()
        ev[1].record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(ev[0].elapsed_time(ev[1]) / R * 1e3)
    print(f"H={Hs} knob {knob}: median {np.median(ts):.2f} us/step")
