import sys, torch
sys.path.insert(0, '/root/repo')
from inputs import TID_K, TID_Q, TID_DO, TID_O_FULL, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
n, H = 8192, 64
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
of = empty_filled(Spec(seed=0, tensor_id=TID_O_FULL, batch=1, n=n, heads=H, d=512))
dh = empty_filled(Spec(seed=0, tensor_id=TID_DO, batch=1, n=n, heads=H, d=512))
a = torch.tensor([0.5], device='cuda'); oh = torch.empty_like(of); osp = torch.empty_like(of)
def t(f, it=10):
    for _ in range(3): f()
    torch.cuda.synchronize(); s, e = torch.cuda.Event(True), torch.cuda.Event(True); s.record()
    for _ in range(it): f()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / it
print("ssa", t(lambda: loza.ssa_prefill(q, kv, out=osp)))
print("fused fwd", t(lambda: loza.ssa_prefill_blend(q, kv, of, a, out=oh)))
print("fused fwd+grad", t(lambda: loza.ssa_prefill_blend(q, kv, of, a, dh, out=oh)))
