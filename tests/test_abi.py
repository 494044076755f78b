"""C-ABI library: loads on a CPU-only host, exports every symbol include/loza.h declares, and validates
arguments on the host before touching the device (no compute calls here)."""
import ctypes
import os
import re

import pytest

from paper_2512_23966_b200 import loza

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "loza.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:loza_status_t|size_t|const char\*|uint64_t|int32_t)\s+(\w+)\s*\(",
                                 src, flags=re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("ssa_prefill", "ssa_decode", "full_attn_ref", "loza_blend", "ssa_seqpar_prefill",
              "ssa_select_blocks"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = loza.lib()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(loza.EXPORTS) == sorted(_declared())


def _args(**kw):
    a = loza.AttnArgs()
    a.batch, a.n_q, a.heads, a.d_qk, a.d_v, a.n_kv = 1, 256, 64, 576, 512, 256
    a.in_dtype = a.out_dtype = loza.LOZA_BF16
    a.softmax_scale, a.causal = 0.1, 1
    a.q = a.k = a.v = a.o = 0x1000
    a.q_stride_b, a.q_stride_tok, a.q_stride_head = 256 * 64 * 576, 64 * 576, 576
    a.k_stride_b, a.k_stride_tok = 256 * 576, 576
    a.v_stride_b, a.v_stride_tok = 256 * 576, 576
    a.o_stride_b, a.o_stride_tok, a.o_stride_head = 256 * 64 * 512, 64 * 512, 512
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("pattern,kw,code", [
    ((1, 0, 128), {}, 1),                       # l < 1
    ((-1, 7, 128), {}, 1),                      # s < 0
    ((1, 7, 0), {}, 1),                         # b < 1
    ((1, 7, 128), {"softmax_scale": float("nan")}, 1),
    ((1, 7, 128), {"causal": 0}, 3),            # SSA is causal only (DESIGN R9)
    ((1, 7, 128), {"causal": 2}, 1),
    ((1, 7, 128), {"n_kv": 100}, 2),            # n_kv < q_start + n_q
    ((1, 7, 128), {"q_start": 64, "n_kv": 512}, 2),  # q_start not a multiple of b
    ((1, 7, 128), {"d_qk": 128, "d_v": 128}, 3),     # bf16 path is the MLA shape only
    ((1, 7, 64), {}, 3),                        # bf16 SSA needs b % 128 == 0
    ((1, 7, 128), {"heads": 0}, 2),
])
def test_host_validation_rejects_before_launch(pattern, kw, code):
    lib = loza.lib()
    a = _args(**kw)
    rc = lib.ssa_prefill(ctypes.byref(a), loza.Pattern(*pattern), None)
    assert rc == code, (rc, lib.loza_last_error())
    assert lib.loza_last_error().decode() != ""


def test_decode_and_blend_validation():
    lib = loza.lib()
    a = _args(n_q=2)
    assert lib.ssa_decode(ctypes.byref(a), ctypes.c_void_p(0x2000), loza.Pattern(1, 7, 128), None, 0, None) == 2
    assert lib.ssa_decode(ctypes.byref(_args(n_q=1)), None, loza.Pattern(1, 7, 128), None, 0, None) == 1
    V = ctypes.c_void_p
    # numel not a multiple of 8
    assert lib.loza_blend(V(16), V(32), V(48), V(64), None, None, 7, 1, None, None, 0, None) == 2
    # d_o_hat without d_alpha
    assert lib.loza_blend(V(16), V(32), V(48), V(64), V(80), None, 8, 1, None, None, 0, None) == 1
    # NULL alpha
    assert lib.loza_blend(V(16), V(32), None, V(64), None, None, 8, 1, None, None, 0, None) == 1
    assert lib.loza_status_string(3) == b"LOZA_ERR_UNSUPPORTED"


def test_seqpar_validation():
    lib = loza.lib()
    a = _args(n_q=256, n_kv=256, q_start=256)
    # world/rank mismatch
    assert lib.ssa_seqpar_prefill(ctypes.byref(a), loza.Pattern(1, 7, 128), None, 2, 2, None, 0, None) == 1
    # shard shorter than the (l-1)*b halo
    assert lib.ssa_seqpar_prefill(ctypes.byref(a), loza.Pattern(1, 7, 128), None, 1, 2, None, 0, None) == 2
    # world > 1 without a communicator
    a2 = _args(n_q=1024, n_kv=1024, q_start=1024)
    assert lib.ssa_seqpar_prefill(ctypes.byref(a2), loza.Pattern(1, 7, 128), None, 1, 2, None, 0, None) == 1
    assert lib.loza_workspace_size(loza.LOZA_WS_SEQPAR, ctypes.byref(a2), loza.Pattern(1, 7, 128), 2) > 0


def _bwd_ws_want(B, n, pat, H=64, slots=74):
    """The backward workspace layout: D [B, n_q*H] fp32, the sink-tile partials
    [B][ceil(s*b/32)][nsplit][32][1088] fp32, the local-tile row-split partials of the pair key kernels
    [B][kt - ns][lsplit][128][1088] fp32 (each region 256-B aligned), then the dS rows [B, n_q*H, (s+l)*b] bf16.
    Row splits: pieces of P whole query blocks, P the smallest <= l (scanning down from l) whose clusters
    B x (sink tiles x ceil(NB/P) + local tiles x ceil(l/P)) fit the cluster slots (148 SMs / 2 without a GPU)."""
    s, l, b = pat
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    kt, nb = -(-n // 128), -(-n // b)
    ns = min(s, kt)
    P = l
    for c in range(l, 0, -1):
        sn = 1 if s == 0 else min(64, -(-nb // c))
        if B * (ns * sn + (kt - ns) * -(-l // c)) > slots:
            break
        P = c
    nsplit = 1 if s == 0 else min(64, -(-nb // P))
    ls = -(-l // P)
    sink = B * -(-min(s * b, n) // 32) * nsplit * 32 * 1088 * 4 if nsplit > 1 else 0
    loc = B * (kt - ns) * ls * 128 * 1088 * 4 if ls > 1 else 0
    return al(B * n * H * 4) + al(sink) + al(loc) + 2 * B * n * H * (s + l) * b


@pytest.mark.parametrize("B,n,pat,want", [
    # 8K: one piece per local tile (P = 7), 10 sink splits
    (2, 8192, (1, 7, 128), 2 * 8192 * 64 * 4 + 2 * 4 * 10 * 32 * 1088 * 4 + 2 * 2 * 8192 * 64 * 1024),
    # 512 tokens: P = 1, every tile split per query block (4 sink splits, 7 local splits)
    (1, 512, (1, 7, 128), 512 * 64 * 4 + 4 * 4 * 32 * 1088 * 4 + 3 * 7 * 128 * 1088 * 4 + 2 * 512 * 64 * 1024),
    (1, 1024, (2, 1, 128), 1024 * 64 * 4 + 8 * 8 * 32 * 1088 * 4 + 2 * 1024 * 64 * 384),  # two sink blocks, 8 splits
    (1, 1024, (0, 2, 128), 1024 * 64 * 4 + 8 * 2 * 128 * 1088 * 4 + 2 * 1024 * 64 * 256),  # no sink blocks, 2 local splits
    (1, 4096, (1, 7, 128), None),  # P = 4
    (3, 2048, (1, 7, 128), None),
    (1, 128, (1, 7, 128), None),  # one block, the sink: no local tiles, no partials
    (1, 256, (2, 7, 128), None),
])
def test_backward_workspace_size(B, n, pat, want):
    """loza_workspace_size(LOZA_WS_BACKWARD) is what attention_backward checks against (host logic only)."""
    a = _args(batch=B, n_q=n, n_kv=n)
    if want is None:
        want = _bwd_ws_want(B, n, pat)
    else:
        assert _bwd_ws_want(B, n, pat) == want
    assert loza.lib().loza_workspace_size(loza.LOZA_WS_BACKWARD, ctypes.byref(a), loza.Pattern(*pat), 1) == want
