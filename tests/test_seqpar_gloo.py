"""Multi-process (gloo, world_size 2 and 4, CPU) check of the sequence-parallel decomposition used by
ssa_seqpar_prefill (csrc/seqpar.cu): rank 0 broadcasts its first s*b KV rows (sink blocks), every rank sends its
last (l-1)*b KV rows to rank+1, and each rank's queries are answered from [sink | halo | shard] alone.

The local attention here is the fp64 oracle restricted to the rows a rank holds after the exchange; it must equal
the oracle over the whole sequence (so the exchange delivers every key the mask allows, and nothing else is
needed). The GPU path of the same exchange is covered bitwise by tests/test_gpu_basic.py (virtual ranks).
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
        s, l, b, n_local, H, d, dv = cfg
        n = n_local * world
        q0 = rank * n_local
        qs = Spec(seed=3, tensor_id=TID_Q, batch=1, n=n, heads=H, d=d, dtype="f32")
        ks = Spec(seed=3, tensor_id=TID_K, batch=1, n=n, heads=1, d=d, dtype="f32")
        vs = Spec(seed=3, tensor_id=TID_V, batch=1, n=n, heads=1, d=dv, dtype="f32")
        k_loc = torch.from_numpy(gen_rows_f32(ks, q0, n_local))
        v_loc = torch.from_numpy(gen_rows_f32(vs, q0, n_local))
        # --- the exchange step (same partition as ssa_seqpar_prefill)
        sink_rows, halo_rows = s * b, (l - 1) * b
        sink_k, sink_v = k_loc[:sink_rows].clone(), v_loc[:sink_rows].clone()
        dist.broadcast(sink_k, src=0)
        dist.broadcast(sink_v, src=0)
        halo_k = torch.zeros(halo_rows, d)
        halo_v = torch.zeros(halo_rows, dv)
        reqs = []
        if halo_rows > 0:
            if rank + 1 < world:
                reqs += [dist.isend(k_loc[n_local - halo_rows:].contiguous(), rank + 1),
                         dist.isend(v_loc[n_local - halo_rows:].contiguous(), rank + 1)]
            if rank > 0:
                reqs += [dist.irecv(halo_k, rank - 1), dist.irecv(halo_v, rank - 1)]
        for r in reqs:
            r.wait()
        # --- rows this rank holds after the exchange, by absolute position
        held = {}
        for j in range(sink_rows):
            held[j] = (sink_k[j].numpy(), sink_v[j].numpy())
        if rank > 0:
            for j in range(halo_rows):
                held[q0 - halo_rows + j] = (halo_k[j].numpy(), halo_v[j].numpy())
        for j in range(n_local):
            held[q0 + j] = (k_loc[j].numpy(), v_loc[j].numpy())
        qf = gen_rows_f32(qs, q0 * H, n_local * H)
        worst = 0.0
        missing = 0
        kf, vf = gen_rows_f32(ks, 0, n), gen_rows_f32(vs, 0, n)  # whole sequence, for the reference only
        for t in range(n_local):
            p = q0 + t
            keys = oracle.allowed_keys(p, n, s, l, b)
            if any(int(j) not in held for j in keys):
                missing += 1
                continue
            kk = np.stack([held[int(j)][0] for j in keys])
            vv = np.stack([held[int(j)][1] for j in keys])
            o_loc, _ = oracle.attend(qf[t * H:(t + 1) * H], kk, vv, 0.4)
            o_ref, _ = oracle.attention_rows(qf[t * H:(t + 1) * H], np.full(H, p), kf, vf, 0.4, s, l, b)
            worst = max(worst, float(np.abs(o_loc - o_ref).max()))
        q_out.put((rank, missing, worst))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [
    (2, (1, 3, 16, 64, 2, 8, 6)),    # (s, l, b, n_local, H, d, dv)
    (4, (1, 7, 8, 64, 1, 4, 4)),     # halo = 6 blocks = 48 rows < shard
    (2, (2, 2, 16, 32, 1, 4, 4)),    # two sink blocks = the whole shard of rank 0
])
def test_seqpar_exchange_gives_every_allowed_key(world, cfg):
    ctx = mp.get_context("spawn")
    qout = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, qout)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [qout.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, missing, worst in res:
        assert missing == 0, f"rank {rank}: {missing} queries need keys outside [sink | halo | shard]"
        assert worst < 1e-12, (rank, worst)
