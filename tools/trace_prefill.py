"""Dump the clock64 timeline of cluster 0 of the prefill kernel (debug hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs import TID_K, TID_Q, Spec
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

mode = sys.argv[1] if len(sys.argv) > 1 else "ssa"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
H = 64
q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=576))
kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=576))
o = torch.empty((1, n, H, 512), dtype=torch.bfloat16, device="cuda")
tr = torch.zeros(22 * 64, dtype=torch.int64, device="cuda")
L = loza.lib()
L.loza_debug_set_trace.argtypes = [ctypes.c_void_p]
if mode in ("calib", "calibf"):  # fused calibration with d_o_hat (ssa_prefill_blend), or forward only
    of = torch.empty_like(o)
    loza.full_attn_ref(q, kv, out=of)
    dh = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=512))
    alpha = torch.tensor([0.5], device="cuda")


def run():
    if mode == "ssa":
        loza.ssa_prefill(q, kv, out=o)
    elif mode == "calib":
        loza.ssa_prefill_blend(q, kv, of, alpha, dh, out=o)
    elif mode == "calibf":
        loza.ssa_prefill_blend(q, kv, of, alpha, out=o)
    else:
        loza.full_attn_ref(q, kv, out=o)


for _ in range(2):
    run()
torch.cuda.synchronize()
L.loza_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
run()
torch.cuda.synchronize()
L.loza_debug_set_trace(ctypes.c_void_p(0))
t = tr.view(22, 64).cpu().numpy().astype("int64")
names = ["S_start", "S_freeok", "S_issued", "PV_start", "PV_pok", "PV_issued", "sm_wait", "sm_sfull", "sm_owait", "sm_ofull", "sm_parr", "kwait", "vwait", "K0_acq", "K4_acq", "V0_acq", "V3_acq"]
base = t[:11][t[:11] > 0].min()
print("tile " + " ".join(f"{x:>9s}" for x in names))
import sys as _s
for g in range(40):
    print(f"{g:4d} " + " ".join(f"{(t[s, g] - base) if t[s, g] > 0 else -1:9d}" for s in range(11)) + f" {t[11, g]:9d} {t[12, g]:9d} "
          + " ".join(f"{(t[s, g] - base) if t[s, g] > 0 else -1:9d}" for s in range(13, 17)))

print("epilogue (unit's last tile g): sm_parr(g) -> O read done -> round0 staged -> round0 read -> round1 staged -> round1 read")
for g in range(40):
    if t[17, g] > 0:
        print(f"{g:4d} parr {t[10, g] - base:9d} oread {t[17, g] - t[10, g]:6d} st0 {t[18, g] - t[17, g]:6d} "
              f"rd0 {t[19, g] - t[18, g]:6d} st1 {t[20, g] - t[19, g]:6d} rd1 {t[21, g] - t[20, g]:6d} "
              f"next_sm_wait {t[6, g + 1] - t[21, g] if g + 1 < 64 else 0:6d}")
