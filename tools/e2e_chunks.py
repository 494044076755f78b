"""e2e (host-resident Q/KV -> device -> SSA prefill -> host O) at 32K vs the number of pipeline chunks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
n, H = 32768, 64
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
qh, kh = q.cpu().pin_memory(), kv.cpu().pin_memory()
qd, kd = torch.empty_like(q), torch.empty_like(kv)
o = torch.empty((1, n, H, 512), dtype=torch.bfloat16, device="cuda")
oh = torch.empty(o.shape, dtype=o.dtype).pin_memory()
s_h, s_c, s_d = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
t = torch.empty(2_000_000_000, dtype=torch.uint8, pin_memory=True)
td = torch.empty(2_000_000_000, dtype=torch.uint8, device="cuda")
ev[0].record(); td.copy_(t, non_blocking=True); ev[1].record(); torch.cuda.synchronize()
print(f"H2D 2 GB: {2e9 / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9:.1f} GB/s")
ev[0].record(); t.copy_(td, non_blocking=True); ev[1].record(); torch.cuda.synchronize()
print(f"D2H 2 GB: {2e9 / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9:.1f} GB/s")
del t, td
for n_chunks in (16, 32, 64):
    nc = n // n_chunks
    eh = [torch.cuda.Event() for _ in range(n_chunks)]
    ec = [torch.cuda.Event() for _ in range(n_chunks)]
    def step():
        cur = torch.cuda.current_stream()
        for s_ in (s_h, s_c, s_d):
            s_.wait_stream(cur)
        for c in range(n_chunks):
            a, e = c * nc, (c + 1) * nc
            with torch.cuda.stream(s_h):
                qd[:, a:e].copy_(qh[:, a:e], non_blocking=True)
                kd[:, a:e].copy_(kh[:, a:e], non_blocking=True)
                eh[c].record(s_h)
            s_c.wait_event(eh[c])
            with torch.cuda.stream(s_c):
                loza.ssa_prefill(qd[:, a:e], kd[:, :e], out=o[:, a:e], q_start=a)
                ec[c].record(s_c)
            s_d.wait_event(ec[c])
            with torch.cuda.stream(s_d):
                oh[:, a:e].copy_(o[:, a:e], non_blocking=True)
        cur.wait_stream(s_d)
        cur.wait_stream(s_c)
    step(); torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        ev[0].record(); step(); ev[1].record(); torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    print(f"chunks {n_chunks}: {np.mean(ts):.2f} ms/step  {n / (np.mean(ts) * 1e-3) / 1e6:.3f} M tok/s")
