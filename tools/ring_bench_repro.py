"""Reproduce the bench's ring-decode row: generator-filled rings vs appended rings, and allocation after
freeing a large cache."""
import sys, torch
sys.path.insert(0, '/root/repo')
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled, fill_
from paper_2512_23966_b200 import loza
B, pat = 64, (1, 7, 128)
big = sys.argv[1] == "big" if len(sys.argv) > 1 else False
if big:
    c = torch.empty((B, 1 << 20, 576), dtype=torch.bfloat16, device='cuda'); del c
q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=64, d=576))
seq = torch.full((B,), 1 << 20, dtype=torch.int32, device='cuda')
rings = []
for r in range(4):
    rc = torch.empty((B, 1024, 576), dtype=torch.bfloat16, device='cuda')
    fill_(rc, Spec(seed=10 + r, tensor_id=TID_K, batch=B, n=1024, heads=1, d=576))
    rings.append(rc)
o = torch.empty((B, 1, 64, 512), dtype=torch.bfloat16, device='cuda')
it = [0]
def fr():
    i = it[0] % 4; it[0] += 1; loza.ssa_decode_ring(q, rings[i], seq, out=o)
fr(); torch.cuda.synchronize()
R = 64
gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(gr, stream=s):
        for _ in range(R): fr()
torch.cuda.synchronize()
for _ in range(2): gr.replay()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
for _ in range(5): gr.replay()
e1.record(); torch.cuda.synchronize(); print("big" if big else "fresh", "generator-filled rings us/step", e0.elapsed_time(e1) / 5 / R * 1e3)
buf = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
ts = []
for _ in range(5):
    buf.fill_(1)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    gr.replay()
    e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) / R * 1e3)
print("with 256 MB flush between replays us/step", sorted(ts))
