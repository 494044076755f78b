"""Small driver for profiling one kernel family (ncu) — not part of the product."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import TID_K, TID_Q, Spec  # noqa: E402
from inputs.device import empty_filled  # noqa: E402
from paper_2512_23966_b200 import loza  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--what", default="ssa", choices=["ssa", "full", "decode", "full_decode", "blend"])
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--ctx", type=int, default=131072)
a = ap.parse_args()
H, dqk = 64, 576
if a.what in ("ssa", "full"):
    q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=a.n, heads=H, d=dqk))
    kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=a.n, heads=1, d=dqk))
    o = torch.empty((1, a.n, H, 512), dtype=torch.bfloat16, device="cuda")
    for _ in range(a.iters):
        if a.what == "ssa":
            loza.ssa_prefill(q, kv, out=o)
        else:
            loza.full_attn_ref(q, kv, out=o)
elif a.what in ("decode", "full_decode"):
    B = 64
    cache = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=B, n=a.ctx, heads=1, d=dqk))
    q = empty_filled(Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=H, d=dqk))
    seq = torch.full((B,), a.ctx, dtype=torch.int32, device="cuda")
    for _ in range(a.iters):
        if a.what == "decode":
            loza.ssa_decode(q, cache, seq)
        else:
            loza.full_attn_ref(q, cache, seq_lens=seq)
torch.cuda.synchronize()
print("probe ok", a.what)
