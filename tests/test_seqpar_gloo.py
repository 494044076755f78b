"""Multi-process (gloo, world_size 2 and 4, CPU) run of the sequence-parallel exchange that ssa_seqpar_prefill
issues (csrc/seqpar.cu), driven by the library's own host plan: every rank asks libloza for its transfer list
(loza_seqpar_plan) and its segmented KV view (loza_seqpar_segments), executes the transfers with
torch.distributed (gloo) on CPU tensors into a workspace laid out exactly as the device workspace, and then
answers each of its queries from [sink | halo | shard] as the library's segments map them.

Checks ("uniform compute across all ranks"; Eq. 4):
- every key the oracle's mask allows for a local query is covered by a segment, and the bytes found there are
  the generator's row of that absolute position (bit for bit) -- the plan delivers the right rows to the right
  offsets, nothing the mask needs is missing;
- the oracle over the gathered rows equals the oracle over the whole sequence (the exchange loses nothing);
- every SEND of rank r matches the RECV of rank r+1 entry for entry, and all ranks list the same broadcasts.
The GPU path of the same plan is covered against the oracle by tests/test_gpu_seqpar.py (virtual ranks and an
NCCL loopback communicator).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from inputs import TID_K, TID_Q, TID_V, Spec, gen_rows_f32


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, q_out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_23966_b200 import loza
        s, l, b, n_local, H, d, dv, B, alias = cfg
        n = n_local * world
        q0 = rank * n_local
        pat = (s, l, b)
        dk = d
        qs = [Spec(seed=3 + bi, tensor_id=TID_Q, batch=1, n=n, heads=H, d=d, dtype="f32") for bi in range(B)]
        ks = [Spec(seed=3 + bi, tensor_id=TID_K, batch=1, n=n, heads=1, d=dk, dtype="f32") for bi in range(B)]
        vs = [Spec(seed=3 + bi, tensor_id=TID_V, batch=1, n=n, heads=1, d=dv, dtype="f32") for bi in range(B)]
        k_loc = [torch.from_numpy(gen_rows_f32(ks[bi], q0, n_local)) for bi in range(B)]
        v_loc = [k_loc[bi][:, :dv] if alias else torch.from_numpy(gen_rows_f32(vs[bi], q0, n_local))
                 for bi in range(B)]
        a = loza.seqpar_host_args(n_local, rank, batch=B, heads=H, d_qk=d, d_v=dv, alias=alias, dtype=loza.LOZA_F32)
        plan = loza.seqpar_plan(a, pat, rank, world)
        segs = loza.seqpar_segments(a, pat, rank, world)
        ws_bytes = loza.lib().loza_workspace_size(loza.LOZA_WS_SEQPAR, a, loza.Pattern(*pat), world)
        ws = torch.zeros(max(ws_bytes, 4) // 4, dtype=torch.float32)

        def own_rows(x):
            src = k_loc[x["batch"]] if x["tensor"] == 0 else v_loc[x["batch"]]
            assert src.shape[1] == x["row_elems"]
            return src[x["src_row"]:x["src_row"] + x["rows"]].contiguous()

        def put(x, t):
            o = x["ws_offset"]
            assert o % 4 == 0 and o + t.numel() * 4 <= ws_bytes
            ws[o // 4:o // 4 + t.numel()] = t.reshape(-1)

        # group 1: sink broadcasts (same list on every rank), group 2: halo sends / receives
        for x in [x for x in plan if x["op"] == loza.XFER_BCAST]:
            buf = own_rows(x) if rank == x["peer"] else torch.empty(x["rows"], x["row_elems"])
            dist.broadcast(buf, src=x["peer"])
            if x["ws_offset"] >= 0:
                put(x, buf)
        reqs, recvd = [], []
        for x in [x for x in plan if x["op"] != loza.XFER_BCAST]:
            if x["op"] == loza.XFER_SEND:
                reqs.append(dist.isend(own_rows(x), x["peer"]))
            else:
                buf = torch.empty(x["rows"], x["row_elems"])
                reqs.append(dist.irecv(buf, x["peer"]))
                recvd.append((x, buf))
        for r in reqs:
            r.wait()
        for x, buf in recvd:
            put(x, buf)

        # the rows each segment maps, by absolute position (the library's own view)
        def ws_row(off, sb, bi, r, elems):
            o = (off + bi * sb) // 4 + r * elems
            return ws[o:o + elems].numpy()

        def key_row(bi, j):
            for g in segs:
                if g["pos_begin"] <= j < g["pos_end"]:
                    r = j - g["pos_begin"]
                    if g["k_off"] < 0:
                        return k_loc[bi][j - q0].numpy(), v_loc[bi][j - q0].numpy()
                    kk = ws_row(g["k_off"], g["k_sb"], bi, r, dk)
                    vv = kk[:dv] if alias else ws_row(g["v_off"], g["v_sb"], bi, r, dv)
                    return kk, vv
            return None

        bad_bytes = missing = 0
        worst = 0.0
        kf = [gen_rows_f32(ks[bi], 0, n) for bi in range(B)]
        vf = [kf[bi][:, :dv] if alias else gen_rows_f32(vs[bi], 0, n) for bi in range(B)]
        for bi in range(B):
            qf = gen_rows_f32(qs[bi], q0 * H, n_local * H)
            for t in range(n_local):
                p = q0 + t
                keys = oracle.allowed_keys(p, n, s, l, b)
                rows = [key_row(bi, int(j)) for j in keys]
                if any(r is None for r in rows):
                    missing += 1
                    continue
                kk = np.stack([r[0] for r in rows])
                vv = np.stack([r[1] for r in rows])
                if not (np.array_equal(kk, kf[bi][keys]) and np.array_equal(vv, vf[bi][keys])):
                    bad_bytes += 1
                o_loc, _ = oracle.attend(qf[t * H:(t + 1) * H], kk, vv, 0.4)
                o_ref, _ = oracle.attention_rows(qf[t * H:(t + 1) * H], np.full(H, p), kf[bi], vf[bi], 0.4, s, l, b)
                worst = max(worst, float(np.abs(o_loc - o_ref).max()))
        q_out.put((rank, missing, bad_bytes, worst, plan))
    finally:
        dist.destroy_process_group()


CASES = [
    # (s, l, b, n_local, H, d, dv, B, v aliases k)
    (2, (1, 3, 16, 64, 2, 8, 6, 1, False)),
    (4, (1, 7, 8, 64, 1, 4, 4, 2, False)),     # halo = 6 blocks = 48 rows < shard; two sequences
    (2, (2, 2, 16, 32, 1, 4, 4, 1, False)),    # two sink blocks = the whole shard of rank 0
    (4, (1, 7, 8, 48, 1, 8, 6, 2, True)),      # MLA aliasing (v = k[:, :dv]); halo = whole previous shard,
                                               # clipped by the sink on rank 1
    (2, (0, 3, 16, 32, 1, 4, 4, 1, True)),     # no sink blocks: halo only
]


@pytest.mark.parametrize("world,cfg", CASES)
def test_seqpar_plan_over_gloo_gives_every_allowed_key(world, cfg):
    ctx = mp.get_context("spawn")
    qout = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, qout)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([qout.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(timeout=60)
    for rank, missing, bad, worst, _ in res:
        assert missing == 0, f"rank {rank}: {missing} queries need keys outside [sink | halo | shard]"
        assert bad == 0, f"rank {rank}: {bad} queries found wrong rows in the exchanged segments"
        assert worst < 1e-12, (rank, worst)
    plans = [r[4] for r in res]
    bc = [[x for x in p if x["op"] == 0] for p in plans]
    for p in bc[1:]:
        assert [(x["batch"], x["tensor"], x["rows"]) for x in p] == [(x["batch"], x["tensor"], x["rows"]) for x in bc[0]]
    for r in range(world - 1):
        sends = [(x["batch"], x["tensor"], x["src_row"], x["rows"], x["row_elems"]) for x in plans[r]
                 if x["op"] == 1]
        recvs = [(x["batch"], x["tensor"], x["src_row"], x["rows"], x["row_elems"]) for x in plans[r + 1]
                 if x["op"] == 2]
        assert sends == recvs
        assert all(x["peer"] == r + 1 for x in plans[r] if x["op"] == 1)
        assert all(x["peer"] == r for x in plans[r + 1] if x["op"] == 2)
