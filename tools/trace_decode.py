"""Dump the clock64 timeline of CTA 0 of the decode kernel (debug hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
B, ctx = 64, int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cache = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=64, d=576))
seq = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
tr = torch.zeros(12 * 32, dtype=torch.int64, device="cuda")
L = loza.lib()
L.loza_debug_set_decode_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    loza.ssa_decode(q, cache, seq)
torch.cuda.synchronize()
L.loza_debug_set_decode_trace(ctypes.c_void_p(tr.data_ptr()))
loza.ssa_decode(q, cache, seq)
torch.cuda.synchronize()
L.loza_debug_set_decode_trace(ctypes.c_void_p(0))
t = tr.view(12, 32).cpu().numpy().astype("int64")
base = t[0, 0]
names = ["setup", "S_start", "S_issued", "PV_start", "PV_pok", "PV_issued", "sm_wait", "sm_sfull", "sm_parr", "piece_end", "part_written", "merge_done"]
for s_ in range(12):
    vals = [int(t[s_, i] - base) if t[s_, i] > 0 else -1 for i in range(8)]
    print(f"{names[s_]:>12s} " + " ".join(f"{v:8d}" for v in vals))
