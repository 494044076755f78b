"""Dump the clock64 timeline of cluster 0 (leader CTA) of the MHA-form prefill kernel (debug hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_K, TID_Q, TID_V, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

sparse = (sys.argv[1] if len(sys.argv) > 1 else "ssa") == "ssa"
n, H = 32768, 64
q, k, v = (empty_filled(Spec(seed=7, tensor_id=t, batch=1, n=n, heads=H, d=d), four_d=True)
           for t, d in ((TID_Q, 192), (TID_K, 192), (TID_V, 128)))
o = torch.empty((1, n, H, 128), dtype=torch.bfloat16, device="cuda")
tr = torch.zeros(10 * 64, dtype=torch.int64, device="cuda")
L = loza.lib()
L.loza_debug_set_trace.argtypes = [ctypes.c_void_p]
for _ in range(2):
    loza.ssa_prefill_mha(q, k, v, out=o, sparse=sparse)
torch.cuda.synchronize()
L.loza_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
loza.ssa_prefill_mha(q, k, v, out=o, sparse=sparse)
torch.cuda.synchronize()
L.loza_debug_set_trace(ctypes.c_void_p(0))
t = tr.view(10, 64).cpu().numpy().astype("int64")
names = ["S_start", "S_ready", "S_issued", "PV_start", "PV_pok", "PV_issued", "sm_sfull", "sm_ofull", "sm_parr", "epi_end"]
base = t[t > 0].min()
print("tile " + " ".join(f"{x:>9s}" for x in names))
for g in range(40):
    print(f"{g:4d} " + " ".join(f"{(t[s, g] - base) if t[s, g] > 0 else -1:9d}" for s in range(10)))
