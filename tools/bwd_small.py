import os, sys
sys.path.insert(0, os.getcwd())
import torch
from inputs import TID_DO, TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
for n, H in ((1152, 8), (640, 16)):
    q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
    kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
    do = empty_filled(Spec(seed=0, tensor_id=TID_DO, batch=1, n=n, heads=H, d=512))
    lse = torch.empty((1, H, n), device="cuda")
    o = loza.ssa_prefill(q, kv, lse=lse)
    dq, dk, dv = loza.attention_backward(q, kv, o, lse, do)
    torch.cuda.synchronize()
    print(n, H, float(dq.abs().sum()), float(dk.abs().sum()), float(dv.abs().sum()))
