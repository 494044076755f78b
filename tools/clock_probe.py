"""Run the headline SSA prefill back to back for a few seconds while sampling SM clock, power and throttle
reasons with nvidia-smi (every 50 ms) - is the kernel power-limited?"""
import os
import subprocess
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

n, H = 32768, 64
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
o = torch.empty((1, n, H, 512), dtype=torch.bfloat16, device="cuda")
what = sys.argv[1] if len(sys.argv) > 1 else "ssa"
fn = (lambda: loza.ssa_prefill(q, kv, out=o)) if what == "ssa" else (lambda: loza.full_attn_ref(q, kv, out=o))
for _ in range(3):
    fn()
torch.cuda.synchronize()
mon = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active,temperature.gpu",
                        "--format=csv,noheader", "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
t0 = time.time()
k = 0
while time.time() - t0 < 4.0:
    for _ in range(20):
        fn()
    k += 20
    torch.cuda.synchronize()
ev[1].record()
torch.cuda.synchronize()
mon.terminate()
lines = mon.communicate()[0].strip().splitlines()
print(f"{what}: {k} launches, {ev[0].elapsed_time(ev[1]) / k:.3f} ms each")
for l in lines[5:-2:8]:
    print(l)
