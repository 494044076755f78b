"""clock64 timeline of one pair cluster of the backward CTA-pair kernels (8K MLA SSA, H64, (1,7,128)):
python tools/trace_bwd.py [mode 1=dV 2=dK] [cluster]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_DO, TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cl = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n = 8192
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=64, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
do = empty_filled(Spec(seed=0, tensor_id=TID_DO, batch=1, n=n, heads=64, d=512))
lse = torch.empty((1, 64, n), device="cuda")
o = loza.ssa_prefill(q, kv, lse=lse)
loza.attention_backward(q, kv, o, lse, do)
torch.cuda.synchronize()
tr = torch.zeros(13 * 2 * 64, dtype=torch.int64, device="cuda")
L = loza.lib()
L.loza_debug_set_bwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
L.loza_debug_set_bwd_trace(ctypes.c_void_p(tr.data_ptr()), cl, mode)
loza.attention_backward(q, kv, o, lse, do)
torch.cuda.synchronize()
L.loza_debug_set_bwd_trace(ctypes.c_void_p(0), 0, 0)
t = tr.view(13, 2, 64).cpu().numpy().astype("int64")
names = ["F_start", "F_sfree", "F_iss", "G_start", "G_pfull", "G_iss", "sm_sfull", "sm_sld", "sm_pdone",
         "sm_pfree", "sm_parr", "ld_first", "ld_grad"]
base = t[t > 0].min()
print("rank tile " + " ".join(f"{x:>9s}" for x in names))
for r in range(2):
    for g in range(24):
        print(f"{r:4d} {g:4d} " + " ".join(f"{(t[s, r, g] - base) if t[s, r, g] > 0 else -1:9d}" for s in range(13)))
