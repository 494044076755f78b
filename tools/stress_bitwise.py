"""Race hunt: repeat the pair backward, the fused calibration and the decode many times and require identical
bits (every kernel here is deterministic by construction). python tools/stress_bitwise.py [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_DO, TID_K, TID_Q, Spec
from inputs.device import empty_filled, fill_
from paper_2512_23966_b200 import loza

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bad = 0
for n, B in ((8192, 1), (2048, 1), (1024, 3)):
    q = empty_filled(Spec(seed=3, tensor_id=TID_Q, batch=B, n=n, heads=64, d=576))
    kv = empty_filled(Spec(seed=3, tensor_id=TID_K, batch=B, n=n, heads=1, d=576))
    do = empty_filled(Spec(seed=3, tensor_id=TID_DO, batch=B, n=n, heads=64, d=512))
    lse = torch.empty((B, 64, n), device="cuda")
    o = loza.ssa_prefill(q, kv, lse=lse)
    ref = [t.clone() for t in loza.attention_backward(q, kv, o, lse, do)]
    for i in range(iters):
        out = loza.attention_backward(q, kv, o, lse, do)
        if not all(torch.equal(a, b) for a, b in zip(out, ref)):
            bad += 1
            print("backward mismatch", n, B, i)
    of = loza.full_attn_ref(q, kv)
    alpha = torch.tensor([0.3], device="cuda")
    b_o, b_d = loza.ssa_prefill_blend(q, kv, of, alpha, do)
    b_o, b_d = b_o.clone(), b_d.clone()
    for i in range(iters):
        o2, d2 = loza.ssa_prefill_blend(q, kv, of, alpha, do)
        if not (torch.equal(o2, b_o) and torch.equal(d2, b_d)):
            bad += 1
            print("calibration mismatch", n, B, i)
    print(f"n={n} B={B}: done", flush=True)
Bd, T = 64, 131072
cache = torch.empty((Bd, T, 576), dtype=torch.bfloat16, device="cuda")
fill_(cache, Spec(seed=4, tensor_id=TID_K, batch=Bd, n=T, heads=1, d=576))
qd = empty_filled(Spec(seed=4, tensor_id=TID_Q, batch=Bd, n=1, heads=64, d=576))
sl = torch.randint(1, T, (Bd,), dtype=torch.int32, device="cuda")
dref = loza.ssa_decode(qd, cache, sl).clone()
for i in range(iters * 10):
    if not torch.equal(loza.ssa_decode(qd, cache, sl), dref):
        bad += 1
        print("decode mismatch", i)
print("mismatches:", bad)
