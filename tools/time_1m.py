"""Time the 1M-token SSA prefill on one GPU (development probe; bench.py carries the official row)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import TID_K, TID_Q, Spec  # noqa: E402
from inputs.device import empty_filled  # noqa: E402
from paper_2512_23966_b200 import loza  # noqa: E402

N, H = 1 << 20, 64
t0 = time.time()
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=N, heads=H, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=N, heads=1, d=576))
o = torch.empty((1, N, H, 512), dtype=torch.bfloat16, device="cuda")
torch.cuda.synchronize()
print("alloc+fill s", time.time() - t0, "free GB", torch.cuda.mem_get_info()[0] / 1e9)
for _ in range(3):
    loza.ssa_prefill(q, kv, out=o)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); loza.ssa_prefill(q, kv, out=o); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
fl = 1006698496 * 139264
print("1M ms", ts, "TFLOP/s", [fl / (t * 1e-3) / 1e12 for t in ts], "Mtok/s", [N / t / 1e3 for t in ts])
