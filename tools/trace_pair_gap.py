"""Gap between two back-to-back pair-decode launches (globaltimer spans of every CTA; debug hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
B, ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 131072
cache = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=64, d=576))
seq = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
L = loza.lib()
L.loza_debug_set_pair_trace.argtypes = [ctypes.c_void_p]
trs = [torch.zeros(12 * 32 + 4 * B, dtype=torch.int64, device="cuda") for _ in range(3)]
for _ in range(3):
    loza.ssa_decode(q, cache, seq)
torch.cuda.synchronize()
for t in trs:
    L.loza_debug_set_pair_trace(ctypes.c_void_p(t.data_ptr()))
    loza.ssa_decode(q, cache, seq)
L.loza_debug_set_pair_trace(ctypes.c_void_p(0))
torch.cuda.synchronize()
sp = [t.cpu().numpy().astype("int64")[12 * 32:].reshape(2 * B, 2) for t in trs]
for i, s in enumerate(sp):
    print(f"launch {i}: first start {s[:, 0].min() - sp[0][:, 0].min():8d} ns, last end {s[:, 1].max() - sp[0][:, 0].min():8d} ns, span {s[:, 1].max() - s[:, 0].min()} ns")
for i in range(1, len(sp)):
    print(f"gap {i - 1}->{i}: {sp[i][:, 0].min() - sp[i - 1][:, 1].max()} ns")
