"""clock64 timeline of cluster 0 of the pair-cooperative decode kernel (debug hook); 'cold' flushes L2 first."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
B, ctx = 64, 131072
cache = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=64, d=576))
seq = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
tr = torch.zeros(11 * 2 * 16 + 32 * B, dtype=torch.int64, device="cuda")
L = loza.lib()
L.loza_debug_set_pair_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
for _ in range(3):
    loza.ssa_decode(q, cache, seq)
torch.cuda.synchronize()
if len(sys.argv) > 1 and sys.argv[1] == "cold":
    fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    fl.fill_(1)
    torch.cuda.synchronize()
L.loza_debug_set_pair_trace(ctypes.c_void_p(tr.data_ptr()), 0)
loza.ssa_decode(q, cache, seq)
torch.cuda.synchronize()
L.loza_debug_set_pair_trace(ctypes.c_void_p(0), 0)
ta = tr.cpu().numpy().astype("int64")
t = ta[:11 * 2 * 16].reshape(11, 2, 16)
sp4 = ta[11 * 2 * 16:11 * 2 * 16 + 16 * B].reshape(2 * B, 8)
wl = ta[11 * 2 * 16 + 16 * B:].reshape(2 * B, 8)
sp = sp4[:, [0, 3]]
names = ["start", "S_start", "S_issued", "PV_start", "PV_pok", "PV_issued", "sm_sfull", "sm_maxsent", "sm_maxok",
         "sm_parr", "end"]
for r in range(2):
    base = t[0, r, 0]
    print(f"--- CTA {r}")
    for s, nm in enumerate(names):
        print(f"{nm:>10s} " + " ".join(f"{(x - base) if x > 0 else -1:7d}" for x in t[s, r, :6]))

import numpy as np
st0 = sp[:, 0].min()
dur = sp[:, 1] - sp[:, 0]
print("per-CTA span ns: min %d median %d max %d; kernel span %d ns; start spread %d ns"
      % (dur.min(), int(np.median(dur)), dur.max(), sp[:, 1].max() - st0, sp[:, 0].max() - st0))
order = np.argsort(-dur)[:8]
print("slowest CTAs:", [(int(i), int(dur[i]), int(sp[i, 0] - st0)) for i in order])

print("phases (ns): start, dep-wait, tiles done, END, after L wait, after last OFull, normalized, before cluster_sync")
for i in list(order[:4]) + list(np.argsort(dur)[:3]):
    print(int(i), [int(x - st0) for x in sp4[i]])

print("per-warp loop exit (ns) of the slowest 2 and fastest 2 CTAs:")
for i in list(order[:2]) + list(np.argsort(dur)[:2]):
    print(int(i), [int(x - st0) for x in wl[i]])
