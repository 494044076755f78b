"""Per-cluster start / end (globaltimer) of the backward CTA-pair kernels: load balance over the grid.
python tools/trace_bwd_clusters.py [mode 1=dV 2=dK] [n]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import TID_DO, TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=64, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
do = empty_filled(Spec(seed=0, tensor_id=TID_DO, batch=1, n=n, heads=64, d=512))
lse = torch.empty((1, 64, n), device="cuda")
o = loza.ssa_prefill(q, kv, lse=lse)
loza.attention_backward(q, kv, o, lse, do)
torch.cuda.synchronize()
kt = n // 128
tr = torch.zeros((kt + 64 * 4) * 2, dtype=torch.int64, device="cuda")  # clusters: local tiles + sink splits
L = loza.lib()
L.loza_debug_set_bwd_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
L.loza_debug_set_bwd_trace(ctypes.c_void_p(tr.data_ptr()), -1, mode)
loza.attention_backward(q, kv, o, lse, do)
torch.cuda.synchronize()
L.loza_debug_set_bwd_trace(ctypes.c_void_p(0), 0, 0)
t = tr.cpu().numpy().reshape(-1, 2)
ok = t[:, 0] > 0
t0 = t[ok, 0].min()
end = t[ok, 1].max()
print(f"kernel span {(end - t0) / 1e3:.1f} us; clusters {ok.sum()} (the sink tiles' row splits first)")
rows = [(i, (t[i, 0] - t0) / 1e3, (t[i, 1] - t0) / 1e3) for i in np.nonzero(ok)[0]]
for pc, s, e in sorted(rows, key=lambda r: r[2]):
    print(f"cluster {pc:4d}: start {s:8.1f} end {e:8.1f} dur {e - s:8.1f} us")
