"""Benchmark of the LoZA SSA hot path on B200 (BASELINE.json metric: SSA prefill & decode tokens/s, % roofline).

Contract (one JSON line on rank 0):
  N=1 : headline workload = BASELINE.json configs[1]: SSA prefill, B1 H64 n32768, MLA-absorbed (576/512),
        (s,l,b) = (1,7,128), bf16 in / fp32 accumulate / bf16 out; value = tokens/s. The other §8 rows
        (full-attention comparator at the same shape, decode B64 at 128K/512K/1M, blend 8K) are measured in
        the same run and reported under "rows".
        The 1M-token SSA prefill on this one GPU (configs[4] at N=1, the base of the strong-scaling curve) is the
        row "ssa_prefill_1m".
  N>1 : sequence-parallel SSA prefill of ONE 1,048,576-token sequence (configs[4]): rank r owns tokens
        [r*2^20/N, (r+1)*2^20/N), NCCL sink broadcast + halo exchange (ssa_seqpar_prefill); strong scaling;
        value = 2^20 tokens / max-rank step time. `python bench.py --gpus N` re-launches itself under
        torch.distributed.run (one process per GPU) when WORLD_SIZE is not set, and fails loudly when the node
        has fewer than N GPUs or WORLD_SIZE disagrees with --gpus.
  --impl reference : the fp64 CPU oracle (oracle/) timed on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PATTERN = (1, 7, 128)
D_QK, D_V, H = 576, 512, 64
N_PREFILL = 32768
N_SP = 1 << 20  # configs[4]: the sequence-parallel prefill's sequence length (all N)
FLOP_PER_PAIR = 2 * (D_QK + D_V) * H  # 139,264


def ssa_pairs(n, s, l, b, q_start=0):
    """Unmasked (query, key) pairs of SSA for queries [q_start, q_start+n): per query block, every earlier
    selected key block (sink blocks kb < s, local blocks qb-l+1 <= kb < qb) gives b keys to each query and the
    own block gives p - qb*b + 1 (DESIGN R2-R5)."""
    tot = 0
    for qb in range(q_start // b, (q_start + n + b - 1) // b):
        lo, hi = max(qb * b, q_start), min((qb + 1) * b, q_start + n)
        prev = len(set(range(min(s, qb))) | set(range(max(0, qb - l + 1), qb)))
        a0, a1 = lo - qb * b + 1, hi - qb * b  # own-block counts of the first / last query
        tot += (hi - lo) * b * prev + (a0 + a1) * (hi - lo) // 2
    return tot


def full_pairs(n):
    return n * (n + 1) // 2


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 5 ms) during the timed region."""

    HW_SLOWDOWN = 0x8
    SW_THERMAL = 0x20
    HW_THERMAL = 0x40
    SW_POWER_CAP = 0x4

    def __init__(self, gpu_index=0, period_s=0.005):
        self.gpu = gpu_index
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, name in ((self.HW_SLOWDOWN, "hw_slowdown"), (self.HW_THERMAL, "hw_thermal_slowdown"),
                                          (self.SW_THERMAL, "sw_thermal_slowdown"), (self.SW_POWER_CAP, "sw_power_cap")):
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(self.period)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "NVML, 5 ms"}


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained"), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def metric_name(world):
    if world == 1:
        return "SSA prefill tokens/s (B1 H64 n32768 MLA 576/512, (s,l,b)=(1,7,128)); % tensor roofline"
    return ("sequence-parallel SSA prefill tokens/s (B1 H64 n1048576 MLA 576/512, (s,l,b)=(1,7,128), "
            f"{world} ranks); % tensor roofline")


def clock_normalized(achieved_tf, sm_mhz, sms=148, flop_per_clk_sm=8192):
    """Achieved algorithmic TFLOP/s over the dense bf16 tcgen05 rate at the SM clock measured during the run
    (148 SMs x 8192 FLOP/clk/SM, B200_PROFILING.md): the tensor-pipe fraction independent of the clock."""
    if not sm_mhz:
        return None
    return achieved_tf / (sms * flop_per_clk_sm * sm_mhz * 1e6 / 1e12)


def _host_available():
    try:
        import psutil
        return float(psutil.virtual_memory().available)
    except Exception:  # noqa: BLE001
        return 0.0


# ----------------------------------------------------------------------------- GPU arm
def _time_events(fn, iters, warmup, flush=None, stream=None):
    """Per-iteration device times (ms) with CUDA events on the launching stream; L2 flushed between iterations."""
    import torch
    stream = stream or torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        if flush is not None:
            flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        fn()
        e.record(stream)
        e.synchronize()
        times.append(s.elapsed_time(e))
    return times


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from inputs import TID_K, TID_Q, Spec
    from inputs.device import empty_filled, fill_
    from paper_2512_23966_b200 import loza

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = measured_peaks()
    scale = loza.default_scale(D_QK)
    s, l, b = PATTERN
    n_total = N_PREFILL if world == 1 else N_SP
    n_local = n_total // world

    # inputs (generated on the device; seed 0, D1 distribution)
    qs = Spec(seed=0, tensor_id=TID_Q, batch=1, n=n_total, heads=H, d=D_QK)
    ks = Spec(seed=0, tensor_id=TID_K, batch=1, n=n_total, heads=1, d=D_QK)
    q = torch.empty((1, n_local, H, D_QK), dtype=torch.bfloat16, device=dev)
    kv = torch.empty((1, n_local, D_QK), dtype=torch.bfloat16, device=dev)
    fill_(q, qs, row_start=rank * n_local * H)
    fill_(kv, ks, row_start=rank * n_local)
    o = torch.empty((1, n_local, H, D_V), dtype=torch.bfloat16, device=dev)
    flush_buf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def flush():
        flush_buf.fill_(1)

    comm_ptr = 0
    if world > 1:
        pg = dist.group.WORLD
        dist.barrier()
        backend = pg._get_backend(dev)
        comm_ptr = backend._comm_ptr()
    ws = None
    if world > 1:
        need = loza.seqpar_ws_bytes(q, kv, kv[..., :D_V], PATTERN, world)
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)

    def step():
        if world == 1:
            loza.ssa_prefill(q, kv, pattern=PATTERN, scale=scale, out=o)
        else:
            loza.ssa_seqpar_prefill(q, kv, pattern=PATTERN, scale=scale, rank=rank, world=world, comm_ptr=comm_ptr,
                                    out=o, ws=ws)

    # ---- headline: K timed steps bracketed by barrier + sync, max over ranks
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = loza.kernel_launches()
    per_step = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            step()
            ev1.record()
            ev1.synchronize()
            per_step.append(ev0.elapsed_time(ev1))
        torch.cuda.synchronize()
    launches = loza.kernel_launches() - launches0
    t_ms = float(np.mean(per_step))
    rank_ms = [t_ms]
    if world > 1:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        allt = [torch.empty_like(tt) for _ in range(world)]
        dist.all_gather(allt, tt)
        rank_ms = [float(x.item()) for x in allt]
        t_ms = max(rank_ms)
    tokens = n_total
    value = tokens / (t_ms * 1e-3)
    pairs = ssa_pairs(n_local, s, l, b, q_start=rank * n_local)
    flops = pairs * FLOP_PER_PAIR
    achieved_tf = flops / (float(np.mean(per_step)) * 1e-3) / 1e12

    rows = {}
    if rank == 0 and world == 1 and not args.quick:
        rows = extra_rows(args, q, kv, o, flush, peaks)
    if world > 1 and not args.quick and not args.no_decode:
        try:
            rows["decode_batch_sharded_128k"] = decode_sharded_leg(world, rank, dev, flush, peaks)
        except Exception as ex:  # noqa: BLE001 -- reported in the line
            rows["decode_batch_sharded_128k"] = {"error": repr(ex)[:300]}

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if world == 1 and not args.no_e2e:
        qh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
        kh = torch.empty(kv.shape, dtype=kv.dtype, pin_memory=True)
        oh = torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
        qh.copy_(q)
        kh.copy_(kv)
        qd = torch.empty_like(q)
        kd2 = [torch.empty_like(kv), torch.empty_like(kv)]  # the KV prefix, double-buffered by step parity

        # Chunked prefill through the public API (q_start = chunk offset, KV prefix up to the chunk's end):
        # chunk c's upload, chunk c-1's SSA and chunk c-2's download overlap on three streams (PCIe is full
        # duplex), and consecutive steps overlap too (a serving pipeline): every step still uploads its own
        # inputs and downloads its own output; per-chunk events keep the reused device buffers safe (Q chunk c:
        # the previous step's SSA of chunk c has read it; O chunk c: the previous step's download has read it;
        # the KV prefix alternates buffers). Units are independent, so the output equals the unchunked
        # prefill bit for bit. Timed as K back-to-back steps between two events (whole-job throughput).
        n_chunks = 32  # 16: 53.0 ms, 32: 50.4 ms, 64: 50.5 ms per step unpipelined (tools/e2e_chunks.py)
        nc = n_local // n_chunks
        s_h, s_c, s_d = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev_h = [torch.cuda.Event() for _ in range(n_chunks)]
        ev_c = [torch.cuda.Event() for _ in range(n_chunks)]
        ev_d = [torch.cuda.Event() for _ in range(n_chunks)]
        ev_step = [torch.cuda.Event(), torch.cuda.Event()]  # SSA of the step with this parity finished
        st_k = [0]

        def e2e_step():
            k = st_k[0]
            st_k[0] += 1
            kd = kd2[k & 1]
            s_h.wait_event(ev_step[k & 1])  # step k-2 (same KV buffer) has finished its SSA
            for c in range(n_chunks):
                a, e = c * nc, (c + 1) * nc
                s_h.wait_event(ev_c[c])  # the previous step's SSA of chunk c has read Q chunk c
                with torch.cuda.stream(s_h):
                    qd[:, a:e].copy_(qh[:, a:e], non_blocking=True)
                    kd[:, a:e].copy_(kh[:, a:e], non_blocking=True)
                    ev_h[c].record(s_h)
                s_c.wait_event(ev_h[c])
                s_c.wait_event(ev_d[c])  # the previous step's download has read O chunk c
                with torch.cuda.stream(s_c):
                    loza.ssa_prefill(qd[:, a:e], kd[:, :e], pattern=PATTERN, scale=scale, out=o[:, a:e], q_start=a)
                    ev_c[c].record(s_c)
                s_d.wait_event(ev_c[c])
                with torch.cuda.stream(s_d):
                    oh[:, a:e].copy_(o[:, a:e], non_blocking=True)
                    ev_d[c].record(s_d)
            ev_step[k & 1].record(s_c)

        cur = torch.cuda.current_stream()
        for _ in range(2):  # warm-up steps
            e2e_step()
        cur.wait_stream(s_d)
        cur.wait_stream(s_c)
        torch.cuda.synchronize()
        k_e2e = max(4, args.steps)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(cur)
        s_h.wait_stream(cur)
        for _ in range(k_e2e):
            e2e_step()
        cur.wait_stream(s_d)
        cur.wait_stream(s_c)
        t1.record(cur)
        t1.synchronize()
        ts = [t0.elapsed_time(t1) / k_e2e]
        # the host copy of the last pipelined step equals the unchunked device prefill bit for bit
        o_ref = loza.ssa_prefill(q, kv, pattern=PATTERN, scale=scale)
        torch.cuda.synchronize()
        e2e_match = bool(torch.equal(oh.to(o_ref.device), o_ref))
        del o_ref
        e2e = {"value": n_local / (float(np.mean(ts)) * 1e-3), "unit": "tokens/s",
               "output_matches_device_prefill": e2e_match,
               "h2d_bytes_per_step": int(q.numel() * 2 + kv.numel() * 2), "d2h_bytes_per_step": int(o.numel() * 2),
               "ms_per_step": float(np.mean(ts)),
               "method": f"ssa_prefill in {n_chunks} chunks (q_start), H2D / compute / D2H on three streams, "
                         f"consecutive steps pipelined; {k_e2e} steps timed back to back"}

    # ---- e2e at N > 1: every rank uploads its shard (pinned host buffers), runs the sequence-parallel
    # prefill through the public API (NCCL sink/halo exchange inside), downloads its output shard; K steps
    # back to back, max over ranks (the same collective sequence on every rank)
    e2e_host_bytes = world * (q.numel() + kv.numel() + o.numel()) * 2  # every rank's pinned shard buffers
    if world > 1 and not args.no_e2e and _host_available() < 1.25 * e2e_host_bytes:
        e2e = {"unavailable": f"needs {e2e_host_bytes / 1e9:.0f} GB of pinned host memory for the {world} ranks' "
                              f"shards, {_host_available() / 1e9:.0f} GB available"}
    elif world > 1 and not args.no_e2e:
        try:
            qh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
            kh = torch.empty(kv.shape, dtype=kv.dtype, pin_memory=True)
            oh = torch.empty(o.shape, dtype=o.dtype, pin_memory=True)
            qh.copy_(q)
            kh.copy_(kv)
            qd, kd = torch.empty_like(q), torch.empty_like(kv)

            def e2e_step_sp():
                qd.copy_(qh, non_blocking=True)
                kd.copy_(kh, non_blocking=True)
                loza.ssa_seqpar_prefill(qd, kd, pattern=PATTERN, scale=scale, rank=rank, world=world,
                                        comm_ptr=comm_ptr, out=o, ws=ws)
                oh.copy_(o, non_blocking=True)

            e2e_step_sp()
            torch.cuda.synchronize()
            dist.barrier()
            k_e2e = max(4, args.steps)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(k_e2e):
                e2e_step_sp()
            t1.record()
            t1.synchronize()
            te = torch.tensor([t0.elapsed_time(t1) / k_e2e], device=dev, dtype=torch.float64)
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            te_ms = float(te.item())
            e2e = {"value": n_total / (te_ms * 1e-3), "unit": "tokens/s",
                   "h2d_bytes_per_step": int(world * (q.numel() + kv.numel()) * 2),
                   "d2h_bytes_per_step": int(world * o.numel() * 2), "ms_per_step": te_ms,
                   "method": "per rank: H2D of its shard, ssa_seqpar_prefill (NCCL exchange), D2H of its output "
                             f"shard; {k_e2e} steps back to back, max over ranks"}
        except Exception as ex:  # noqa: BLE001 -- reported in the line, the headline still prints
            e2e = {"error": repr(ex)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_seconds, n_total)

    if rank == 0:
        frac = achieved_tf / peaks["bf16_tflops"]
        csum = clk.summary()
        line = {
            "metric": metric_name(world),
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms, "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
            "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (counter-based N(0,1)-like, seed 0; inputs/gen.py)",
            "config": {"workload": "ssa_prefill_32k" if world == 1 else "ssa_seqpar_prefill_1m",
                       "batch": 1, "seq_len": n_total, "tokens_per_gpu": n_local, "heads": H, "d_qk": D_QK,
                       "d_v": D_V, "pattern": list(PATTERN), "softmax_scale": scale,
                       "parallelism": f"sp{world}" if world > 1 else "single",
                       "l2": "flushed between timed steps (256 MB write)" if world == 1 else
                             "flushed between timed steps (256 MB write); per-rank inputs (>= 9.7 GB) exceed L2"},
            "per_rank_ms": rank_ms,
            "roofline": {"bound": "tensor", "kernel": "prefill_tc_kernel", "achieved": achieved_tf,
                         "peak": peaks["bf16_tflops"], "unit": "TFLOP/s", "frac": frac,
                         "clock_normalized_frac": clock_normalized(achieved_tf, csum.get("sm_mhz")),
                         "traffic": ncu_traffic("prefill_tc_kernel") if world == 1 else None,
                         "traffic_note": "DRAM bytes per launch from the committed ncu capture (profiles/); "
                                         "algorithmic Q+KV+O bytes = 4.60e9",
                         "algorithmic_flop_per_launch": flops, "pairs_per_launch": pairs,
                         "peak_source": peaks["source"] + " bf16_tflops (burst)",
                         "frac_vs_sustained": achieved_tf / peaks["bf16_tflops_sustained"]
                         if peaks.get("bf16_tflops_sustained") else None},
            "clocks": csum,
            "gpu_launches": int(launches),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "rows": rows,
            "paper_context": {"decode_ssa_vs_flashmla_128k": ">=90% less cost (PAPER.md:244, hardware unstated)",
                              "e2e_prefill_speedup_256k": ">50% (PAPER.md:244)",
                              "e2e_decode_saving_256k": ">30% (PAPER.md:244)"},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def extra_rows(args, q, kv, o, flush, peaks):
    """The other §8 rows, each with its own roofline: full prefill comparator, decode (128K/512K/1M), blend 8K."""
    import torch

    from inputs import TID_DO, TID_K, TID_Q, Spec
    from inputs.device import fill_
    from paper_2512_23966_b200 import loza
    out = {}
    scale = loza.default_scale(D_QK)
    dev = q.device
    if not args.no_1m:
        try:
            out["ssa_prefill_1m"] = prefill_1m_row(peaks, flush)
        except Exception as e:  # noqa: BLE001 -- reported in the line
            out["ssa_prefill_1m"] = {"error": repr(e)[:300]}
        torch.cuda.empty_cache()
    # full-attention prefill at the same shape
    t = _time_events(lambda: loza.full_attn_ref(q, kv, scale=scale, out=o), 2, 1, flush)
    fl = full_pairs(N_PREFILL) * FLOP_PER_PAIR
    tf = fl / (float(np.mean(t)) * 1e-3) / 1e12
    out["full_prefill_32k"] = {"ms": float(np.mean(t)), "tokens_per_s": N_PREFILL / (np.mean(t) * 1e-3),
                               "tflops": tf, "frac_tensor": tf / peaks["bf16_tflops"]}
    # blend at 8K (configs[2]): full + SSA forward, blend + d_alpha
    n8 = 8192
    q8, kv8 = q[:, :n8], kv[:, :n8]
    of = torch.empty((1, n8, H, D_V), dtype=torch.bfloat16, device=dev)
    osp = torch.empty_like(of)
    dh = torch.empty_like(of)
    fill_(dh, Spec(seed=0, tensor_id=TID_DO, batch=1, n=n8, heads=H, d=D_V))
    alpha = torch.tensor([0.5], device=dev)
    oh = torch.empty_like(of)
    dal = torch.empty(1, dtype=torch.float64, device=dev)
    t_full = _time_events(lambda: loza.full_attn_ref(q8, kv8, scale=scale, out=of), 3, 1, flush)
    t_ssa = _time_events(lambda: loza.ssa_prefill(q8, kv8, pattern=PATTERN, scale=scale, out=osp), 10, 2, flush)
    t_bl = _time_events(lambda: loza.loza_blend(of, osp, alpha, dh, out=oh, d_alpha=dal), 10, 3, flush)
    bl_bytes = of.numel() * 2 * 4
    out["blend_8k"] = {"full_ms": float(np.mean(t_full)), "ssa_ms": float(np.mean(t_ssa)),
                       "blend_ms": float(np.mean(t_bl)),
                       "blend_gbs": bl_bytes / (np.mean(t_bl) * 1e-3) / 1e9,
                       "blend_frac_hbm": bl_bytes / (np.mean(t_bl) * 1e-3) / 1e9 / peaks["hbm_gbs"],
                       "ssa_frac_tensor": ssa_pairs(n8, *PATTERN) * FLOP_PER_PAIR / (np.mean(t_ssa) * 1e-3) / 1e12
                       / peaks["bf16_tflops"],
                       "full_frac_tensor": full_pairs(n8) * FLOP_PER_PAIR / (np.mean(t_full) * 1e-3) / 1e12
                       / peaks["bf16_tflops"]}
    # fused calibration forward: SSA + Eq. 3 + d_alpha in one kernel (O' never stored)
    t_fu = _time_events(lambda: loza.ssa_prefill_blend(q8, kv8, of, alpha, dh, pattern=PATTERN, scale=scale, out=oh),
                        10, 2, flush)
    t_ff = _time_events(lambda: loza.ssa_prefill_blend(q8, kv8, of, alpha, pattern=PATTERN, scale=scale, out=oh),
                        10, 2, flush)
    t_bf = _time_events(lambda: loza.loza_blend(of, osp, alpha, out=oh), 10, 3, flush)
    fu_ms = float(np.mean(t_fu))
    out["calibration_fused_8k"] = {
        "fused_ms": fu_ms, "unfused_ms": float(np.mean(t_ssa)) + float(np.mean(t_bl)),
        "speedup_vs_unfused": (float(np.mean(t_ssa)) + float(np.mean(t_bl))) / fu_ms,
        "fused_fwd_only_ms": float(np.mean(t_ff)), "unfused_fwd_only_ms": float(np.mean(t_ssa)) + float(np.mean(t_bf)),
        "speedup_fwd_only_vs_unfused": (float(np.mean(t_ssa)) + float(np.mean(t_bf))) / float(np.mean(t_ff)),
        "ssa_frac_tensor_in_fused": ssa_pairs(n8, *PATTERN) * FLOP_PER_PAIR / (fu_ms * 1e-3) / 1e12
        / peaks["bf16_tflops"],
        "note": "unfused = ssa_prefill (writes O') + loza_blend with d_alpha (reads O, O', dO_hat; writes O_hat)"}
    # attention backward at the same 8K shape: SSA gradients of Q and the latent KV
    lse8 = torch.empty((1, H, n8), device=dev)
    loza.ssa_prefill(q8, kv8, pattern=PATTERN, scale=scale, out=osp, lse=lse8)
    t_bw = _time_events(lambda: loza.attention_backward(q8, kv8, osp, lse8, dh, pattern=PATTERN, scale=scale),
                        5, 2, flush)
    bw_ms = float(np.mean(t_bw))
    bw_flop = ssa_pairs(n8, *PATTERN) * H * 2 * (3 * D_QK + 2 * D_V)  # recompute S, dP, dQ, dK, dV
    out["backward_ssa_8k"] = {
        "ms": bw_ms, "tflops": bw_flop / (bw_ms * 1e-3) / 1e12,
        "frac_tensor": bw_flop / (bw_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
        "kernel": "tcgen05 (attn_bwd_tc.cu: D beside the dV kernel; 128-key CTA-pair dV kernel (cta_group::2, S three "
                  "row tiles ahead, P halves swapped by bulk DSMEM copies, dV^T in TMEM, P into the dS rows) and dK kernel "
                  "(P from the dS rows, dK^T in TMEM, dS rows); dQ = dS K GEMM; sink tiles split by query blocks + "
                  "fixed-order reduce); the 64-key kernels 4.25 ms, the 32-key one-pass key kernel 6.1 ms, warp-MMA 22 ms, "
                  "FFMA 492 ms before it",
        "algorithmic_flop": bw_flop}
    del of, osp, dh, oh
    # non-absorbed (MHA-form) SSA prefill: per-head K/V (192 / 128) at the headline's 32K
    from inputs import TID_V
    qm, km, vm = (torch.empty((1, N_PREFILL, H, d), dtype=torch.bfloat16, device=dev) for d in (192, 192, 128))
    for t_, tid in ((qm, TID_Q), (km, TID_K), (vm, TID_V)):
        fill_(t_, Spec(seed=0, tensor_id=tid, batch=1, n=N_PREFILL, heads=H, d=t_.shape[-1]))
    om = torch.empty((1, N_PREFILL, H, 128), dtype=torch.bfloat16, device=dev)
    t_m = _time_events(lambda: loza.ssa_prefill_mha(qm, km, vm, PATTERN, out=om), 5, 2, flush)
    t_mf = _time_events(lambda: loza.ssa_prefill_mha(qm, km, vm, out=om, sparse=False), 2, 1, flush)
    mha_fl = ssa_pairs(N_PREFILL, *PATTERN) * H * 2 * (192 + 128)
    mha_ffl = full_pairs(N_PREFILL) * H * 2 * (192 + 128)
    m_ms, mf_ms = float(np.mean(t_m)), float(np.mean(t_mf))
    out["mha_ssa_prefill_32k"] = {
        "ms": m_ms, "tokens_per_s": N_PREFILL / (m_ms * 1e-3), "tflops": mha_fl / (m_ms * 1e-3) / 1e12,
        "frac_tensor": mha_fl / (m_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
        "full_ms": mf_ms, "full_tflops": mha_ffl / (mf_ms * 1e-3) / 1e12,
        "full_frac_tensor": mha_ffl / (mf_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
        "ssa_vs_full": mf_ms / m_ms,
        "shape": "B1, 32768 tokens, H64, q/k 192, v 128 per head, (1,7,128); K/V up-projection not included",
        "algorithmic_flop": mha_fl}
    del qm, km, vm, om
    if not args.no_cpu:
        try:
            ot = oracle_row_timings()
            out["oracle_beside_rows"] = ot
        except Exception as e:  # noqa: BLE001
            out["oracle_beside_rows"] = {"error": repr(e)[:200]}
    # decode B64 at 128K / 512K / 1M (configs[3])
    if not args.no_decode:
        try:
            out["decode"] = decode_rows(args, peaks, flush)
        except Exception as e:  # report, do not hide: the headline line still prints
            out["decode"] = {"error": repr(e)[:300]}
    return out


def prefill_1m_row(peaks, flush, steps=5, warmup=2):
    """configs[4] on ONE GPU: SSA prefill of a 1,048,576-token sequence (B1 H64 MLA 576/512, (1,7,128)): Q 77.3 GB,
    O 68.7 GB bf16 (the base of the strong-scaling curve of the N>1 lines; parity: tests/test_gpu_1m.py).
    A step is ~0.14 s of continuous tensor work, so the clock settles under the power cap: the roofline is
    given against the SUSTAINED bf16 peak (MEASURED_PEAKS.json) and clock-normalised."""
    import torch

    from inputs import TID_K, TID_Q, Spec
    from inputs.device import empty_filled
    from paper_2512_23966_b200 import loza
    n = N_SP
    need = n * H * (D_QK + D_V) * 2 + n * D_QK * 2
    free = torch.cuda.mem_get_info()[0]
    if free < need + (1 << 30):
        return {"skipped": f"needs {need / 1e9:.1f} GB of device memory, {free / 1e9:.1f} GB free"}
    q = empty_filled(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=D_QK))
    kv = empty_filled(Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=D_QK))
    o = torch.empty((1, n, H, D_V), dtype=torch.bfloat16, device=q.device)
    scale = loza.default_scale(D_QK)
    with ClockSampler(q.device.index) as clk:
        t = _time_events(lambda: loza.ssa_prefill(q, kv, pattern=PATTERN, scale=scale, out=o), steps, warmup, flush)
    del q, kv, o
    ms = float(np.mean(t))
    fl = ssa_pairs(n, *PATTERN) * FLOP_PER_PAIR
    tf = fl / (ms * 1e-3) / 1e12
    c = clk.summary()
    sus = peaks.get("bf16_tflops_sustained") or peaks["bf16_tflops"]
    return {"ms": ms, "ms_all": t, "tokens_per_s": n / (ms * 1e-3),
            "roofline": {"bound": "tensor", "kernel": "prefill_tc_kernel", "achieved": tf, "unit": "TFLOP/s",
                         "peak": sus, "frac": tf / sus, "peak_source": peaks["source"] + " bf16_tflops_sustained",
                         "frac_vs_burst": tf / peaks["bf16_tflops"],
                         "clock_normalized_frac": clock_normalized(tf, c.get("sm_mhz")),
                         "algorithmic_flop_per_launch": fl, "pairs_per_launch": ssa_pairs(n, *PATTERN)},
            "clocks": c, "steps": steps, "warmup": warmup,
            "config": {"workload": "ssa_prefill_1m", "batch": 1, "seq_len": n, "heads": H, "pattern": list(PATTERN),
                       "l2": "inputs (146 GB) exceed L2; flushed between steps anyway"}}


def time_decode_graph(q, cache, seqs, outs, flush, R=64):
    """Per-step time (ms) of ssa_decode captured R times in one CUDA graph over rotating windows/outputs (a serving
    engine graph-captures the decode step), L2 flushed before each replay; median of 5 replays."""
    import torch

    from paper_2512_23966_b200 import loza
    scale = loza.default_scale(D_QK)
    for r in range(len(seqs)):  # warm-up (also initialises the decode workspace outside the capture)
        loza.ssa_decode(q, cache, seqs[r], pattern=PATTERN, scale=scale, out=outs[r])
    torch.cuda.synchronize()
    gs = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(gs, stream=cs):
            for i in range(R):
                loza.ssa_decode(q, cache, seqs[i % len(seqs)], pattern=PATTERN, scale=scale, out=outs[i % len(outs)])
    torch.cuda.synchronize()
    tg = _time_events(lambda: gs.replay(), 5, 2, flush)
    return float(np.median(tg)) / R


def decode_sharded_leg(world, rank, dev, flush, peaks):
    """Decode sharded by batch at N > 1 (SURVEY.md §8 e; no collective): every rank decodes its own 64 sequences
    at 128K context (weak scaling: 64 sequences per GPU); value = all ranks' sequences / max-rank step time."""
    import torch
    import torch.distributed as dist

    from inputs import TID_K, TID_Q, Spec
    from inputs.device import fill_
    B, ctx = 64, 131072
    cache = torch.empty((B, ctx, D_QK), dtype=torch.bfloat16, device=dev)
    fill_(cache, Spec(seed=0, tensor_id=TID_K, batch=B * world, n=ctx, heads=1, d=D_QK), row_start=rank * B * ctx)
    q = torch.empty((B, 1, H, D_QK), dtype=torch.bfloat16, device=dev)
    fill_(q, Spec(seed=1, tensor_id=TID_Q, batch=B * world, n=1, heads=H, d=D_QK), row_start=rank * B * H)
    seqs = [torch.full((B,), ctx - 2048 * r, dtype=torch.int32, device=dev) for r in range(4)]
    outs = [torch.empty((B, 1, H, D_V), dtype=torch.bfloat16, device=dev) for _ in range(4)]
    ms = time_decode_graph(q, cache, seqs, outs, flush)
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    by = world * B * (1024 * D_QK * 2 + H * D_QK * 2 + H * D_V * 2)
    del cache
    return {"ssa_us_per_step": ms * 1e3, "sequences_per_gpu": B, "context": ctx,
            "tokens_per_s": world * B / (ms * 1e-3), "gbs_all_ranks": by / (ms * 1e-3) / 1e9,
            "frac_hbm_per_gpu": by / world / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"], "scaling": "weak",
            "timing": "CUDA graph of 64 steps, 4 rotating windows, max over ranks"}


def decode_rows(args, peaks, flush):
    import torch

    from inputs import TID_K, TID_Q, Spec
    from inputs.device import fill_
    from paper_2512_23966_b200 import loza
    dev = torch.device("cuda", torch.cuda.current_device())
    B = 64
    free = torch.cuda.mem_get_info()[0]
    t_cap = 1 << 20
    while B * t_cap * D_QK * 2 > free * 0.8 and t_cap > (1 << 17):
        t_cap //= 2
    cache = torch.empty((B, t_cap, D_QK), dtype=torch.bfloat16, device=dev)
    fill_(cache, Spec(seed=0, tensor_id=TID_K, batch=B, n=t_cap, heads=1, d=D_QK))
    qd = torch.empty((B, 1, H, D_QK), dtype=torch.bfloat16, device=dev)
    fill_(qd, Spec(seed=1, tensor_id=TID_Q, batch=B, n=1, heads=H, d=D_QK))
    od = torch.empty((B, 1, H, D_V), dtype=torch.bfloat16, device=dev)
    scale = loza.default_scale(D_QK)
    res = {}
    ws = None
    # decode over the bounded ring cache (measured first, before the full-attention
    # comparators heat the GPU): (s+l)*b rows per sequence (75 MB at B=64) filled
    # from the window of a 1M-token sequence; 4 rotating caches (300 MB > L2) in the graph
    R_rows = (PATTERN[0] + PATTERN[1]) * PATTERN[2]
    ctx_ring = 1048576
    rings = []
    for r in range(4):
        rc = torch.empty((B, R_rows, D_QK), dtype=torch.bfloat16, device=dev)
        fill_(rc, Spec(seed=10 + r, tensor_id=TID_K, batch=B, n=R_rows, heads=1, d=D_QK))
        rings.append(rc)
    seq = torch.full((B,), ctx_ring, dtype=torch.int32, device=dev)
    outs = [torch.empty((B, 1, H, D_V), dtype=torch.bfloat16, device=dev) for _ in range(4)]
    for r in range(4):
        loza.ssa_decode_ring(qd, rings[r], seq, pattern=PATTERN, scale=scale, out=outs[r])
    torch.cuda.synchronize()
    R = 64
    gs = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(gs, stream=cs):
            for i in range(R):
                loza.ssa_decode_ring(qd, rings[i % 4], seq, pattern=PATTERN, scale=scale, out=outs[i % 4])
    torch.cuda.synchronize()
    tg = _time_events(lambda: gs.replay(), 5, 2, flush)
    ms = float(np.median(tg)) / R
    by = B * (R_rows * D_QK * 2 + H * D_QK * 2 + H * D_V * 2)
    res["ring_1048576"] = {"ssa_us": ms * 1e3, "ssa_tokens_per_s": B / (ms * 1e-3), "ssa_gbs": by / (ms * 1e-3) / 1e9,
                           "ssa_frac_hbm": by / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                           "cache_bytes": B * R_rows * D_QK * 2,
                           "note": "bounded ring cache (s+l)*b rows per sequence, position 1M; bitwise equal to the "
                                   "contiguous-cache decode (tests/test_ring_cache.py)"}
    del rings
    for ctx in (131072, 524288, 1048576):
        if ctx > t_cap:
            continue
        # 4 rotating windows (seq_len = ctx, ctx - 2048, ...) so consecutive steps do not hit in L2
        # (84 MB per step vs 126 MB L2); R steps captured in one CUDA graph so host launch overhead
        # is not timed (a serving engine graph-captures the decode step).
        seqs = [torch.full((B,), ctx - 2048 * r, dtype=torch.int32, device=dev) for r in range(4)]
        outs = [torch.empty((B, 1, H, D_V), dtype=torch.bfloat16, device=dev) for _ in range(4)]
        R = 64
        ms = time_decode_graph(qd, cache, seqs, outs, flush, R)
        window = min(ctx, (PATTERN[0] + PATTERN[1]) * PATTERN[2])
        by = B * (window * D_QK * 2 + H * D_QK * 2 + H * D_V * 2)
        res[str(ctx)] = {"ssa_us": ms * 1e3, "ssa_tokens_per_s": B / (ms * 1e-3), "ssa_gbs": by / (ms * 1e-3) / 1e9,
                         "ssa_frac_hbm": by / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                         "ssa_bytes": by, "ssa_timing": f"CUDA graph of {R} steps, 4 rotating windows"}
    # decode sharded by heads (north star; SURVEY.md §8 e "if B < R"): one GPU's share of a head-sharded decode,
    # B64 with H/2 = 32 heads over the same latent windows (the pair-cooperative kernel with zero-padded heads,
    # attn_tc_decode_coop.cu); per-GPU bytes hardly drop (the window is shared by all heads)
    if "131072" in res:
        ctx, Hs = 131072, 32
        qh = qd[:, :, :Hs].contiguous()
        seqs = [torch.full((B,), ctx - 2048 * r, dtype=torch.int32, device=dev) for r in range(4)]
        outs = [torch.empty((B, 1, Hs, D_V), dtype=torch.bfloat16, device=dev) for _ in range(4)]
        ms = time_decode_graph(qh, cache, seqs, outs, flush)
        by = B * (1024 * D_QK * 2 + Hs * D_QK * 2 + Hs * D_V * 2)
        res["heads32_131072"] = {"ssa_us": ms * 1e3, "ssa_tokens_per_s": B / (ms * 1e-3),
                                 "ssa_gbs": by / (ms * 1e-3) / 1e9,
                                 "ssa_frac_hbm": by / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                                 "kernel": "pair-cooperative, heads 32..63 zero-padded (attn_tc_decode_coop.cu)",
                                 "note": "B64, 32 of 64 heads: one GPU of a 2-way head-sharded decode"}
    # full-attention comparators after every SSA row (their long max-bandwidth runs heat the GPU and slowed
    # SSA rows timed right after them by up to 30%)
    for ctx in (131072, 524288, 1048576):
        if str(ctx) not in res:
            continue
        seq0 = torch.full((B,), ctx, dtype=torch.int32, device=dev)
        tf = lambda: loza.full_attn_ref(qd, cache, scale=scale, seq_lens=seq0, out=od)  # noqa: E731
        tfull = _time_events(tf, 3, 1, flush)
        by_full = B * (ctx * D_QK * 2 + H * D_QK * 2 + H * D_V * 2)
        res[str(ctx)].update({"full_ms": float(np.mean(tfull)),
                              "full_gbs": by_full / (np.mean(tfull) * 1e-3) / 1e9,
                              "full_frac_hbm": by_full / (np.mean(tfull) * 1e-3) / 1e9 / peaks["hbm_gbs"],
                              "ssa_cost_vs_full": res[str(ctx)]["ssa_us"] * 1e-3 / float(np.mean(tfull))})
    del cache
    return res


# ----------------------------------------------------------------------------- CPU oracle arm
def cpu_baseline(seconds: float = 15.0, n: int = N_PREFILL):
    """The fp64 oracle, as it stands, on a bounded sample of the headline workload: all 64 heads of random
    query tokens of the n-token SSA prefill ((1,7,128)). Per token the oracle derives the allowed keys from its
    own mask (oracle.allowed_keys) and attends over exactly those rows (oracle.attend); only those two calls
    are timed (the rows are regenerated from the counter-based generator outside the timer).
    Returns tokens/s of the oracle."""
    import oracle
    from inputs import TID_K, TID_Q, Spec, gen_rows_f32
    qs = Spec(seed=0, tensor_id=TID_Q, batch=1, n=n, heads=H, d=D_QK)
    ks = Spec(seed=0, tensor_id=TID_K, batch=1, n=n, heads=1, d=D_QK)
    rng = np.random.default_rng(0)
    done, t0 = 0, time.perf_counter()
    spent = 0.0
    s, l, b = PATTERN
    kf = gen_rows_f32(ks, 0, n) if n <= 65536 else None  # whole KV once when small (75 MB at 32K)
    while spent < seconds:
        for t in np.sort(rng.integers(0, n, 8)):
            t = int(t)
            qr = gen_rows_f32(qs, t * H, H)
            lo = max(0, (t // b - l + 1) * b)
            if kf is None:  # the rows the window can touch: sink blocks and the local blocks
                rows = np.concatenate([np.arange(min(s * b, lo)), np.arange(lo, t + 1)])
                kw = np.concatenate([gen_rows_f32(ks, 0, min(s * b, lo)), gen_rows_f32(ks, lo, t + 1 - lo)])
            ta = time.perf_counter()
            keys = oracle.allowed_keys(t, n, s, l, b)
            kk = kf[keys] if kf is not None else kw[np.searchsorted(rows, keys)]
            oracle.attend(qr, kk, kk[:, :D_V], loza_scale())
            spent += time.perf_counter() - ta
            done += 1
    wall = time.perf_counter() - t0
    return {"value": done / spent, "unit": "tokens/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{done} random query tokens x 64 heads of the {n}-token SSA prefill (fp64, OpenMP over "
                      f"rows; oracle.allowed_keys + oracle.attend per token); {spent:.1f} s of oracle time "
                      f"({wall:.1f} s wall incl. input regeneration)",
            "oracle_s": spent, "wall_s": wall, "cpu_model": _cpu_model()}


def oracle_row_timings(seconds_each: float = 1.5):
    """The fp64 oracle timed beside the extra rows, each on a bounded sample extrapolated to the row's
    workload (host cores, OpenMP). Returns {row: {...}}."""
    import oracle
    from inputs import TID_DO, TID_K, TID_Q, Spec, gen_rows_f32
    out = {}
    scale = loza_scale()
    ks = Spec(seed=0, tensor_id=TID_K, batch=1, n=2048, heads=1, d=D_QK)
    qs = Spec(seed=0, tensor_id=TID_Q, batch=1, n=2048, heads=H, d=D_QK)
    kf = gen_rows_f32(ks, 0, 2048)
    # decode: one sequence's step = 64 heads over the 1,024-key window
    win = kf[:1024]
    qr = gen_rows_f32(qs, 0, H)
    n_it, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds_each:
        oracle.attend(qr, win, np.ascontiguousarray(win[:, :D_V]), scale)
        n_it += 1
    per_seq = (time.perf_counter() - t0) / n_it
    out["decode"] = {"oracle_ms_per_step_b64": per_seq * 64 * 1e3, "sample": f"{n_it} sequences (64 heads x 1024 keys)"}
    # blend: elements per second
    x = np.random.default_rng(0).standard_normal(1 << 22).astype(np.float32)
    n_it, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds_each:
        oracle.blend(x, x, 0.5, x)
        n_it += 1
    el_s = n_it * x.size / (time.perf_counter() - t0)
    out["blend_8k"] = {"oracle_ms": 8192 * H * D_V / el_s * 1e3, "sample": f"{n_it} x 4M elements (Eq. 3 + d_alpha)"}
    # backward: (row, key) pairs per second on a 256-token SSA problem, extrapolated to the 8K row
    n_b = 256
    qb = gen_rows_f32(qs, 0, n_b * H)
    dos = Spec(seed=0, tensor_id=TID_DO, batch=1, n=n_b, heads=H, d=D_V)
    dob = gen_rows_f32(dos, 0, n_b * H)
    pos = np.repeat(np.arange(n_b), H)
    t0 = time.perf_counter()
    oracle.attention_backward(qb, pos, kf[:n_b], np.ascontiguousarray(kf[:n_b, :D_V]), dob, scale, *PATTERN)
    dt = time.perf_counter() - t0
    pairs_small = sum(min(t + 1, 1024) for t in range(n_b)) * H  # (1,7,128) window covers all of 256 tokens
    out["backward_ssa_8k"] = {"oracle_ms": dt / pairs_small * ssa_pairs(8192, *PATTERN) * H * 1e3,
                              "sample": f"{n_b} tokens x 64 heads, full backward (two passes)"}
    # MHA-form SSA: one head, 1024 query rows against their (1,7,128) windows, extrapolated to 32K x 64 heads
    n_m = 1024
    qh = gen_rows_f32(Spec(seed=0, tensor_id=TID_Q, batch=1, n=n_m, heads=1, d=192), 0, n_m)
    kh = gen_rows_f32(Spec(seed=0, tensor_id=TID_K, batch=1, n=n_m, heads=1, d=192), 0, n_m)
    vh = np.ascontiguousarray(kh[:, :128])
    t0 = time.perf_counter()
    oracle.attention_rows(qh, np.arange(n_m), kh, vh, 1.0 / np.sqrt(192.0), *PATTERN)
    dt = time.perf_counter() - t0
    out["mha_ssa_prefill_32k"] = {"oracle_ms": dt / ssa_pairs(n_m, *PATTERN) * ssa_pairs(N_PREFILL, *PATTERN) * H
                                  * 1e3, "sample": f"{n_m} tokens x 1 head (d 192 / 128)"}
    return out


def loza_scale():
    return 1.0 / math.sqrt(192.0)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    """--impl reference: the fp64 oracle as it stands, on the host cores, on the GPU arm's config and metric
    (N=1: the 32K prefill; N>1: the 1M-token sequence-parallel prefill). Each step is a bounded sample of that
    workload; value = sampled tokens / oracle seconds. ms_per_step is the wall time a step actually took;
    projected_full_step_ms is the oracle's time for the whole step at the sampled rate (a projection)."""
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_total = N_PREFILL if world == 1 else N_SP
    per, walls = [], []
    cb = None
    for _ in range(args.warmup):
        cpu_baseline(min(2.0, args.cpu_seconds), n_total)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(args.cpu_seconds / max(1, args.steps) * 2, n_total)
        walls.append(time.perf_counter() - t0)
        per.append(cb["value"])
    value = float(np.mean(per))
    line = {"impl": "reference",
            "metric": metric_name(world),
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(walls)) * 1e3,  # measured: one bounded sample per step
            "projected_full_step_ms": n_total / value * 1e3,  # projection: the whole step at the sampled rate
            "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (counter-based, seed 0)",
            "config": {"workload": "ssa_prefill_32k" if world == 1 else "ssa_seqpar_prefill_1m", "batch": 1,
                       "seq_len": n_total, "heads": H, "pattern": list(PATTERN)},
            "cpu_baseline": {"kind": "oracle", "cores": cb["cores"], "sample": cb["sample"], "value": value,
                             "unit": "tokens/s"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _relaunch_distributed(n):
    """`bench.py --gpus N` without WORLD_SIZE: re-run this command under torch.distributed.run, one process per
    GPU (NCCL_DEBUG=INFO so the rank count of the communicator is in the log). Fails loudly when the node has
    fewer than N GPUs -- never a silent 1-GPU run."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        sys.stderr.write(f"bench.py: --gpus {n} needs {n} visible GPUs, this node has {have}\n")
        sys.exit(2)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true", help="headline only (no extra rows)")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-1m", action="store_true", help="skip the 1M-token single-GPU prefill row")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None and int(ws_env) != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ws_env} but --gpus {args.gpus}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and ws_env is None:
        _relaunch_distributed(args.gpus)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
