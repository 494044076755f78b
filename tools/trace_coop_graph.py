"""Per-step globaltimer phases of the pair-cooperative decode inside the bench's CUDA graph (B64 at 128K,
4 rotating windows, L2 flushed before the replay): every captured step writes its own trace buffer, so the
steady state (start spread, head, tile phase, tail, gap to the next step) is visible."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from inputs import TID_K, TID_Q, Spec
from inputs.device import fill_
from paper_2512_23966_b200 import loza

B, ctx, H, P = 64, 131072, 64, (1, 7, 128)
R = int(os.environ.get("STEPS", "16"))
cache = torch.empty((B, ctx, 576), dtype=torch.bfloat16, device="cuda")
fill_(cache, Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
qd = torch.empty((B, 1, H, 576), dtype=torch.bfloat16, device="cuda")
fill_(qd, Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=H, d=576))
seqs = [torch.full((B,), ctx - 2048 * r, dtype=torch.int32, device="cuda") for r in range(4)]
outs = [torch.empty((B, 1, H, 512), dtype=torch.bfloat16, device="cuda") for _ in range(4)]
NT = 11 * 2 * 16 + 32 * B
trs = [torch.zeros(NT, dtype=torch.int64, device="cuda") for _ in range(R)]
L = loza.lib()
L.loza_debug_set_pair_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
for r in range(4):
    loza.ssa_decode(qd, cache, seqs[r], pattern=P, out=outs[r])
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
with torch.cuda.stream(cs):
    with torch.cuda.graph(g, stream=cs):
        for i in range(R):
            L.loza_debug_set_pair_trace(ctypes.c_void_p(trs[i].data_ptr()), 0)
            loza.ssa_decode(qd, cache, seqs[i % 4], pattern=P, out=outs[i % 4])
L.loza_debug_set_pair_trace(ctypes.c_void_p(0), 0)
torch.cuda.synchronize()
fl = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(3):
    fl.fill_(it)
    ev[0].record()
    g.replay()
    ev[1].record()
    torch.cuda.synchronize()
print(f"graph: {ev[0].elapsed_time(ev[1]) / R * 1e3:.2f} us/step (traced build)")
sp = [t.cpu().numpy().astype(np.int64)[11 * 2 * 16:11 * 2 * 16 + 16 * B].reshape(2 * B, 8) for t in trs]
t00 = sp[0][:, 0].min()
print("step: min start, max start, median(after wait, tiles done, L wait, OFull, normalized, pre-sync, end), max end "
      "(ns from the step's first CTA start); gap = this step's first start - previous step's last end")
prev_end = None
for i, s in enumerate(sp):
    st = s[:, 0].min()
    rel = s - st
    med = [int(np.median(rel[:, k])) for k in (1, 2, 4, 5, 6, 7, 3)]
    gap = (st - prev_end) if prev_end is not None else 0
    print(f"{i:3d} t0 {st - t00:8d}  start {int(rel[:, 0].min()):5d}..{int(rel[:, 0].max()):5d}  "
          f"med {med}  end max {int(rel[:, 3].max()):6d}  gap {gap:6d}")
    prev_end = s[:, 3].max()

names = ["start", "S_start", "S_issued", "PV_start", "PV_pok", "PV_issued", "sm_sfull", "sm_maxsent", "sm_maxok",
         "sm_parr", "end"]
for i in (R // 2, R - 1):
    t = trs[i].cpu().numpy().astype(np.int64)[:11 * 2 * 16].reshape(11, 2, 16)
    print(f"--- step {i}, cluster 0, clock64 cycles from CTA 0's post-wait stamp")
    for r in range(2):
        base = t[0, 0, 0]
        print(f"  CTA {r}")
        for s, nm in enumerate(names):
            print(f"  {nm:>10s} " + " ".join(f"{(x - base) if x > 0 else -1:7d}" for x in t[s, r, :(8 if nm == 'end' else 6)]))
