"""How much host-side launch latency lands inside the bench's device timing: the 32K prefill timed with and without a
spin kernel ahead of the start event (python tools/host_gap.py)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import fill_
from paper_2512_23966_b200 import loza
n, H = 32768, 64
q = torch.empty((1, n, H, 576), dtype=torch.bfloat16, device="cuda"); fill_(q, Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
kv = torch.empty((1, n, 576), dtype=torch.bfloat16, device="cuda"); fill_(kv, Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
o = torch.empty((1, n, H, 512), dtype=torch.bfloat16, device="cuda")
fb = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
step = lambda: loza.ssa_prefill(q, kv, pattern=(1, 7, 128), out=o)
for _ in range(3): step()
torch.cuda.synchronize()
def run(sleep):
    ts = []
    for _ in range(20):
        fb.fill_(1)
        if sleep: torch.cuda._sleep(sleep)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); step(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return np.mean(ts), np.min(ts)
import time
t0 = time.perf_counter(); [loza.ssa_prefill(q, kv, pattern=(1, 7, 128), out=o) for _ in range(0)]; 
for s in (0, 1_000_000, 0, 1_000_000):
    print(s, run(s))
# host overhead of one call
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(50):
    torch.cuda._sleep(10_000_000)
    step()
t1 = time.perf_counter(); print("host us per call (queued behind sleeps):", (t1 - t0) / 50 * 1e6)
torch.cuda.synchronize()
