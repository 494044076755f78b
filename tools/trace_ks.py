"""clock64 timeline of cluster 0 of the key-split decode kernel (attn_tc_decode_ks.cu, KTRACE slots)."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import fill_
from paper_2512_23966_b200 import loza

B, ctx, H, P = 64, 131072, 64, (1, 7, 128)
cache = torch.empty((B, ctx, 576), dtype=torch.bfloat16, device="cuda")
fill_(cache, Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
qd = torch.empty((B, 1, H, 576), dtype=torch.bfloat16, device="cuda")
fill_(qd, Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=H, d=576))
seq = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
out = torch.empty((B, 1, H, 512), dtype=torch.bfloat16, device="cuda")
tr = torch.zeros(9 * 2 * 32, dtype=torch.int64, device="cuda")
lib = loza.lib()
lib.loza_debug_set_ks_trace.argtypes = [ctypes.c_void_p]
for i in range(3):
    lib.loza_debug_set_ks_trace(ctypes.c_void_p(tr.data_ptr() if i == 2 else 0))
    tr.zero_()
    fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); fl.fill_(1)
    loza.ssa_decode(qd, cache, seq, pattern=P, out=out)
    torch.cuda.synchronize()
t = tr.view(9, 2, 32).cpu().numpy().astype("int64")
names = ["start/wait", "TMA issue", "MMA S issue", "MMA PV issue", "SM sfull", "SM redor", "SM exact", "SM pfull",
         "merge"]
for r in range(2):
    base = t[0, r, 0]
    print(f"--- CTA {r}")
    for sl in range(9):
        vals = [int(v - base) if v else None for v in t[sl, r]]
        vals = [v for v in vals if v is not None]
        print(f"{names[sl]:14s}", " ".join(f"{v:6d}" for v in vals[:12]))
