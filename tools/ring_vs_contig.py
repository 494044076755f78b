"""Decode over the ring cache vs the contiguous cache on identical rows (graph-timed, no L2 flush)."""
import sys, torch
sys.path.insert(0, '/root/repo')
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
B, ctx, pat = 64, int(sys.argv[1]) if len(sys.argv) > 1 else 131072, (1, 7, 128)
cache = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=B, n=ctx, heads=1, d=576))
q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=64, d=576))
seq = torch.full((B,), ctx, dtype=torch.int32, device='cuda')
ring = torch.zeros((B, 1024, 576), dtype=torch.bfloat16, device='cuda')
loza.ssa_ring_append(ring, cache, torch.zeros(B, dtype=torch.int32, device='cuda'), pattern=pat)
o1 = loza.ssa_decode(q, cache, seq); o2 = loza.ssa_decode_ring(q, ring, seq)
torch.cuda.synchronize(); print("bitwise equal:", torch.equal(o1, o2))
def g(f, R=64):
    f(); torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            for _ in range(R): f()
    torch.cuda.synchronize()
    for _ in range(2): gr.replay()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True); e0.record()
    for _ in range(5): gr.replay()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 5 / R * 1e3
print("contig us/step", g(lambda: loza.ssa_decode(q, cache, seq, out=o1)))
print("ring   us/step", g(lambda: loza.ssa_decode_ring(q, ring, seq, out=o2)))
# rotating: 4 windows of the contiguous cache vs 4 separate ring caches (the bench's methodology)
seqs = [torch.full((B,), ctx - 2048 * r, dtype=torch.int32, device='cuda') for r in range(4)]
rings = []
for r in range(4):
    rr = torch.zeros((B, 1024, 576), dtype=torch.bfloat16, device='cuda')
    loza.ssa_ring_append(rr, cache[:, :ctx - 2048 * r], torch.zeros(B, dtype=torch.int32, device='cuda'), pattern=pat)
    rings.append(rr)
it = [0]
def fc():
    i = it[0] % 4; it[0] += 1; loza.ssa_decode(q, cache, seqs[i], out=o1)
def fr():
    i = it[0] % 4; it[0] += 1; loza.ssa_decode_ring(q, rings[i], seqs[i], out=o2)
print("rotating contig us/step", g(fc))
print("rotating ring   us/step", g(fr))
