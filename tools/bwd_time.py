"""One SSA backward call at the bench shape (8K, H64, MLA, (1,7,128)) for launch-list timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_DO, TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
knob = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # loza_debug_force_kernel("backward", knob)
if knob:
    loza.lib().loza_debug_force_kernel(b"backward", knob)
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=64, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
do = empty_filled(Spec(seed=0, tensor_id=TID_DO, batch=1, n=n, heads=64, d=512))
lse = torch.empty((1, 64, n), device="cuda")
o = loza.ssa_prefill(q, kv, lse=lse)
loza.attention_backward(q, kv, o, lse, do)  # warm-up (module load, attributes)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for i in range(3):
    ev[i].record()
    loza.attention_backward(q, kv, o, lse, do)
ev[3].record()
torch.cuda.synchronize()
ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
print(f"backward n={n} (knob {knob}): " + " ".join(f"{t:.2f}" for t in ts) + " ms")
