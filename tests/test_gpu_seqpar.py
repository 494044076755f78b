"""Sequence-parallel SSA prefill (SURVEY.md §8 a10 / e; north star "halo exchange of the l local blocks + sink
broadcast") on the GPU, checked against the fp64 ORACLE over the whole sequence.

One GPU runs every rank ("virtual ranks", the only multi-rank form allowed on one GPU: no kernel waits on another
rank's kernel). The shard's exchange is the library's plan (loza_seqpar_plan) executed either by device copies
(loza_seqpar_prefill_local) or through REAL NCCL calls on a one-rank communicator from torch's ProcessGroupNCCL
(loza_seqpar_prefill_loopback: ncclBroadcast / ncclSend + ncclRecv with the same counts, datatypes and offsets
ssa_seqpar_prefill issues). Then the split launch: the interior query blocks over [sink | shard] while the halo is
in flight, the first l-1 blocks over [sink | halo | shard] after it.

Rows at risk: each shard's first l-1 blocks (they read the halo), the sink rows seen from rank > 0,
the shard boundaries, the halo clipped by the sink (rank 1 when the halo spans the whole previous shard), and the
LSE of the split launch (its head stride is the shard's n_q). Tolerance (DESIGN R12): bf16 max-abs <= 2e-2 with a
1e-2 normwise guard, LSE 1e-3 relative; fp32 path normwise 1e-4.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
from inputs import TID_K, TID_Q, TID_V, Spec, gen_rows_f32
from inputs.device import empty_filled
from paper_2512_23966_b200 import loza

pytestmark = pytest.mark.gpu

H, D_QK, D_V = 64, 576, 512


def _specs(seed, B, n, kind):
    qk = "q_sink" if kind == "sink" else "plain"
    kk = {"sink": "kv_sink", "marker": "kv_marker"}.get(kind, "plain")
    qs = Spec(seed=seed, tensor_id=TID_Q, batch=B, n=n, heads=H, d=D_QK, kind=qk, amp=5.27, col=D_QK - 1)
    ks = Spec(seed=seed, tensor_id=TID_K, batch=B, n=n, heads=1, d=D_QK, kind=kk,
              amp=5.27 if kind == "sink" else 0.5, col=D_QK - 1, sink_rows=128, block=128, marker_mod=D_V)
    return qs, ks


def _run_virtual(q, kv, world, pat, mode, comm_ptr=0, with_lse=True):
    B, n = q.shape[0], q.shape[1]
    nl = n // world
    shards = [kv[:, r * nl:(r + 1) * nl].contiguous() for r in range(world)]
    outs, lses = [], []
    for r in range(world):
        qr = q[:, r * nl:(r + 1) * nl].contiguous()
        lse = torch.full((B, H, nl), float("nan"), device="cuda") if with_lse else None
        kw = dict(rank=r, world=world, rank0_k=shards[0], prev_k=shards[r - 1] if r > 0 else None, lse=lse)
        if mode == "local":
            o = loza.ssa_seqpar_prefill_local(qr, shards[r], None, pat, loza.default_scale(D_QK), **kw)
        else:
            o = loza.ssa_seqpar_prefill_loopback(qr, shards[r], None, pat, loza.default_scale(D_QK),
                                                 comm_ptr=comm_ptr, **kw)
        outs.append(o)
        lses.append(lse)
    torch.cuda.synchronize()
    return torch.cat(outs, 1), (torch.cat(lses, 2) if with_lse else None)


def _check_oracle(o, lse, qs, ks, pat, toks):
    s, l, b = pat
    n = qs.n
    scale = loza.default_scale(D_QK)
    for bi in range(qs.batch):
        kf = gen_rows_f32(ks, bi * n, n)
        for t in toks:
            qr = gen_rows_f32(qs, (bi * n + t) * H, H)
            ref, rl = oracle.attention_rows(qr, np.full(H, t), kf, kf[:, :D_V], scale, s, l, b)
            got = o[bi, t].double().cpu().numpy()
            err = np.abs(got - ref).max()
            assert err <= 2e-2, (bi, t, err)
            assert err / np.abs(ref).max() <= 1e-2, (bi, t, err)
            if lse is not None:
                gl = lse[bi, :, t].double().cpu().numpy()
                assert np.abs(gl - rl).max() <= 1e-3 * max(1.0, np.abs(rl).max()), (bi, t)


def _risky_tokens(world, nl, l, b):
    toks = set()
    for r in range(world):
        base = r * nl
        for off in (0, 1, b - 1, b, (l - 1) * b - 1, (l - 1) * b, nl - 1):
            if 0 <= off < nl:
                toks.add(base + off)
    return sorted(toks)


@pytest.mark.parametrize("world,nl,kind,B", [
    (4, 1024, "marker", 1),   # halo 768 rows inside the previous shard
    (4, 768, "marker", 2),    # halo = the whole previous shard; rank 1's halo clipped by the sink; 2 sequences
    (2, 1024, "sink", 1),     # sink-heavy data (~50% of the mass on block 0), seen from rank 1
    (8, 896, "plain", 1),
])
def test_seqpar_virtual_ranks_vs_oracle(world, nl, kind, B):
    pat = (1, 7, 128)
    n = world * nl
    qs, ks = _specs(71 + world, B, n, kind)
    q, kv = empty_filled(qs), empty_filled(ks)
    o, lse = _run_virtual(q, kv, world, pat, "local")
    assert not torch.isnan(lse).any().item()
    _check_oracle(o, lse, qs, ks, pat, _risky_tokens(world, nl, 7, 128))
    # and bit for bit the one-GPU prefill (units are computed the same way in every launch)
    ref = loza.ssa_prefill(q, kv, pattern=pat)
    torch.cuda.synchronize()
    assert torch.equal(o, ref)


def test_seqpar_pattern_2_3_vs_oracle():
    """Two sink blocks and l = 3 (halo 2 blocks), 4 ranks of 512 tokens."""
    pat, world, nl = (2, 3, 128), 4, 512
    qs, ks = _specs(75, 1, world * nl, "marker")
    q, kv = empty_filled(qs), empty_filled(ks)
    o, lse = _run_virtual(q, kv, world, pat, "local")
    _check_oracle(o, lse, qs, ks, pat, _risky_tokens(world, nl, 3, 128))


def test_seqpar_fp32_separate_v_vs_oracle():
    """fp32 SIMT path with a separate V (the plan moves k and v rows), d 64, (1, 3, 32), 4 ranks."""
    pat, world, nl, d = (1, 3, 32), 4, 64, 64
    n = world * nl
    qs = Spec(seed=76, tensor_id=TID_Q, batch=1, n=n, heads=2, d=d, dtype="f32")
    ks = Spec(seed=76, tensor_id=TID_K, batch=1, n=n, heads=1, d=d, dtype="f32")
    vs = Spec(seed=76, tensor_id=TID_V, batch=1, n=n, heads=1, d=d, dtype="f32")
    q, k, v = empty_filled(qs), empty_filled(ks), empty_filled(vs)
    ksh = [k[:, r * nl:(r + 1) * nl].contiguous() for r in range(world)]
    vsh = [v[:, r * nl:(r + 1) * nl].contiguous() for r in range(world)]
    kf, vf = gen_rows_f32(ks, 0, n), gen_rows_f32(vs, 0, n)
    for r in range(world):
        lse = torch.full((1, 2, nl), float("nan"), device="cuda")
        o = loza.ssa_seqpar_prefill_local(q[:, r * nl:(r + 1) * nl].contiguous(), ksh[r], vsh[r], pat, 0.125,
                                          rank=r, world=world, rank0_k=ksh[0], rank0_v=vsh[0],
                                          prev_k=ksh[r - 1] if r > 0 else None,
                                          prev_v=vsh[r - 1] if r > 0 else None, lse=lse)
        torch.cuda.synchronize()
        qf = gen_rows_f32(qs, r * nl * 2, nl * 2)
        ref, rl = oracle.attention_rows(qf, np.repeat(np.arange(r * nl, (r + 1) * nl), 2), kf, vf, 0.125, *pat)
        got = o[0].double().cpu().numpy().reshape(-1, d)
        assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-4, r
        gl = lse[0].double().cpu().numpy().T.reshape(-1)
        assert np.abs(gl - rl).max() <= 1e-5 * max(1.0, np.abs(rl).max()), r


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_comm():
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev)
    t = torch.ones(1, device=dev)
    dist.all_reduce(t)  # creates the communicator
    torch.cuda.synchronize()
    ptr = dist.group.WORLD._get_backend(dev)._comm_ptr()
    assert ptr != 0
    yield ptr
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nl,B", [(4, 1024, 1), (4, 768, 2), (2, 896, 1)])
def test_seqpar_nccl_loopback_vs_oracle(nccl_comm, world, nl, B):
    """The exchange through real NCCL calls (one-rank communicator): bitwise equal to the one-GPU prefill and
    in tolerance against the oracle on the risky rows."""
    pat = (1, 7, 128)
    n = world * nl
    qs, ks = _specs(81 + world + B, B, n, "marker")
    q, kv = empty_filled(qs), empty_filled(ks)
    o, lse = _run_virtual(q, kv, world, pat, "loopback", comm_ptr=nccl_comm)
    ref_lse = torch.empty((B, H, n), device="cuda")
    ref = loza.ssa_prefill(q, kv, pattern=pat, lse=ref_lse)
    torch.cuda.synchronize()
    assert torch.equal(o, ref)
    assert torch.equal(lse, ref_lse)
    _check_oracle(o, lse, qs, ks, pat, _risky_tokens(world, nl, 7, 128)[::2])


def test_seqpar_real_entry_point_world1(nccl_comm):
    """ssa_seqpar_prefill itself at world 1 (no exchange: one launch) equals ssa_prefill bitwise."""
    pat, n = (1, 7, 128), 2048
    qs, ks = _specs(90, 1, n, "plain")
    q, kv = empty_filled(qs), empty_filled(ks)
    o = loza.ssa_seqpar_prefill(q, kv, pattern=pat, rank=0, world=1, comm_ptr=nccl_comm)
    ref = loza.ssa_prefill(q, kv, pattern=pat)
    torch.cuda.synchronize()
    assert torch.equal(o, ref)
