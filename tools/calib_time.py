"""The bench's fused-calibration row (8K, B1, H64, (1,7,128), alpha 0.5, L2 flushed before each call):
python tools/calib_time.py  (LOZA_LIB=... to time a variant)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs import TID_DO, TID_K, TID_Q, Spec
from inputs.device import empty_filled, fill_
from paper_2512_23966_b200 import loza

n, H, pat = 8192, 64, (1, 7, 128)
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
of = torch.empty((1, n, H, 512), dtype=torch.bfloat16, device="cuda")
osp, dh, oh = torch.empty_like(of), torch.empty_like(of), torch.empty_like(of)
fill_(dh, Spec(seed=0, tensor_id=TID_DO, batch=1, n=n, heads=H, d=512))
alpha = torch.tensor([0.5], device="cuda")
dal = torch.empty(1, dtype=torch.float64, device="cuda")
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
loza.full_attn_ref(q, kv, out=of)


def t(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    out = []
    for _ in range(iters):
        flush_buf.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


ssa = t(lambda: loza.ssa_prefill(q, kv, pattern=pat, out=osp))
bl = t(lambda: loza.loza_blend(of, osp, alpha, dh, out=oh, d_alpha=dal))
blf = t(lambda: loza.loza_blend(of, osp, alpha, out=oh))
fu = t(lambda: loza.ssa_prefill_blend(q, kv, of, alpha, dh, pattern=pat, out=oh))
ff = t(lambda: loza.ssa_prefill_blend(q, kv, of, alpha, pattern=pat, out=oh))
print(f"calib 8K: fused+dalpha {fu:.3f} ms vs unfused {ssa + bl:.3f} ({(ssa + bl) / fu:.3f}x); "
      f"fwd-only {ff:.3f} vs {ssa + blf:.3f} ({(ssa + blf) / ff:.3f}x); ssa {ssa:.3f}")
