import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
B, ctx = 64, 131072
cache = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=64, d=576))
seq = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
tr = torch.zeros(12 * 32 + 2 * 2 * B + 64, dtype=torch.int64, device="cuda")
L = loza.lib()
L.loza_debug_set_pair_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    loza.ssa_decode(q, cache, seq)
torch.cuda.synchronize()
L.loza_debug_set_pair_trace(ctypes.c_void_p(tr.data_ptr()))
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if len(sys.argv) > 1 and sys.argv[1] == "cold":  # flush L2 so the traced step streams from HBM (as in the bench)
    fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    fl.fill_(1)
    torch.cuda.synchronize()
s.record(); loza.ssa_decode(q, cache, seq); e.record()
torch.cuda.synchronize()
print("event time (us, incl. host launch gap)", s.elapsed_time(e) * 1e3)
L.loza_debug_set_pair_trace(ctypes.c_void_p(0))
ta = tr.cpu().numpy().astype("int64")
t = ta[:12 * 32].reshape(12, 32)
sp = ta[12 * 32:12 * 32 + 4 * B].reshape(2 * B, 2)
kw = ta[12 * 32 + 4 * B:12 * 32 + 4 * B + 32]
vw = ta[12 * 32 + 4 * B + 32:]
print('ring waits in S per tile', kw[:6], ' in PV', vw[:6])
base = t[0, 0]
for nm, row in zip(["setup", "S_start", "S_issued", "PV_start", "PV_pok", "PV_issued", "sm_wait", "sm_sfull", "sm_parr", "piece_end", "merge_sent", "done"], t):
    print(f"{nm:>10s} " + " ".join(f"{(x - base) if x > 0 else -1:7d}" for x in row[:9]))

st0 = sp[:, 0].min()
dur = sp[:, 1] - sp[:, 0]
print("per-CTA span ns: min %d median %d max %d; kernel span (first start -> last end) %d ns; start spread %d ns"
      % (dur.min(), int(np.median(dur)), dur.max(), sp[:, 1].max() - st0, sp[:, 0].max() - st0))
