"""Relative errors of the SSA backward against the fp64 oracle for small shapes: python tools/bwd_small_check.py [knob]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from inputs import TID_DO, TID_K, TID_Q, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza
knob = int(sys.argv[1]) if len(sys.argv) > 1 else 0
if knob:
    loza.lib().loza_debug_force_kernel(b"backward", knob)
for n, Hh, pat in ((257, 8, (1, 7, 128)), (200, 1, (1, 2, 128)), (130, 64, (1, 7, 128)), (256, 8, (1, 7, 128)),
                   (384, 8, (1, 7, 128)), (300, 8, (1, 1, 128)), (1152, 8, (1, 7, 128))):
    qs = Spec(seed=93, tensor_id=TID_Q, batch=1, n=n, heads=Hh, d=576)
    ks = Spec(seed=93, tensor_id=TID_K, batch=1, n=n, heads=1, d=576)
    dos = Spec(seed=93, tensor_id=TID_DO, batch=1, n=n, heads=Hh, d=512)
    q, kv, do = empty_filled(qs), empty_filled(ks), empty_filled(dos)
    scale = loza.default_scale(576)
    kf = gen_rows_f32(ks, 0, n)
    orow, lrow = oracle.attention_rows(gen_rows_f32(qs, 0, n * Hh), np.repeat(np.arange(n), Hh), kf, kf[:, :512],
                                       scale, *pat, sparse=True, causal=True)
    o = torch.from_numpy(orow.reshape(1, n, Hh, 512)).to(torch.bfloat16).cuda()
    lse = torch.from_numpy(lrow.reshape(n, Hh).T.copy()[None]).float().cuda()
    dq, dk, dv = loza.attention_backward(q, kv, o, lse, do, pattern=pat, scale=scale)
    torch.cuda.synchronize()
    rq, rk, rv = oracle.attention_backward(gen_rows_f32(qs, 0, n * Hh), np.repeat(np.arange(n), Hh), kf, kf[:, :512],
                                           gen_rows_f32(dos, 0, n * Hh), scale, *pat, sparse=True, causal=True)
    e = lambda g, r: np.linalg.norm(g - r) / max(np.linalg.norm(r), 1e-30)  # noqa: E731
    gk, gv = dk[0].double().cpu().numpy(), dv[0].double().cpu().numpy()
    bad = [j for j in range(n) if np.linalg.norm(gk[j] - rk[j]) > 0.05 * max(np.linalg.norm(rk[j]), 1e-9)]
    print(f"n={n} H={Hh} pat={pat}: dq {e(dq[0].reshape(-1, 576).double().cpu().numpy(), rq):.2e} "
          f"dk {e(gk, rk):.2e} dv {e(gv, rv):.2e}  bad keys {bad[:10]} ({len(bad)})")
