"""A/B timer for the headline SSA prefill (32K, H64, MLA, (1,7,128)) with an L2 flush between launches.
Run once per library build: LOZA_LIB=variants/libloza_X.so python tools/ab_ssa.py [iters]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n, H = 32768, 64
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
o = torch.empty((1, n, H, 512), dtype=torch.bfloat16, device="cuda")
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for i in range(iters + 3):
    fl.fill_(i & 0xff)
    ev[0].record()
    loza.ssa_prefill(q, kv, out=o)
    ev[1].record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(ev[0].elapsed_time(ev[1]))
ts = np.array(ts)
print(f"{os.environ.get('LOZA_LIB', 'default'):40s} median {np.median(ts):.4f} ms  mean {ts.mean():.4f}  min {ts.min():.4f}")
