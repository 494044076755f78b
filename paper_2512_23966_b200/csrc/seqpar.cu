// Sequence-parallel SSA prefill (north star; SURVEY.md §8 a10 / e).
//
// Each rank owns a contiguous, block-aligned shard [q_start, q_start + n_local)
// of one long sequence (all ranks equal: PAPER.md:89, layer-level sparsity gives
// every rank the same schedule). A query block needs its s sink blocks (rank 0's
// first s*b rows) and its l local blocks; only the first l-1 blocks of a shard
// reach back into the previous rank's last (l-1)*b rows. So one exchange step
// suffices, issued as ONE NCCL group on the caller's stream:
//   ncclBroadcast(sink rows, root 0)  +  ncclSend(last (l-1)*b rows -> r+1)
//                                     +  ncclRecv(halo <- r-1)
// followed by the local SSA prefill over the segmented KV [sink | halo | shard].
// The output stays sharded; no gather, no LSE merge.
//
// NCCL is resolved at run time from the libnccl.so.2 already loaded by the
// caller's process (torch), so the communicator from ProcessGroupNCCL's
// _comm_ptr() is used with the very library that created it.
#include <dlfcn.h>
#include <string.h>

#include <nccl.h>

#include "internal.h"

namespace loza {

namespace {

struct NcclApi {
  ncclResult_t (*group_start)();
  ncclResult_t (*group_end)();
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  const char* (*err)(ncclResult_t);
  bool ok;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return a;
    a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
    a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
    a.send = (decltype(a.send))dlsym(h, "ncclSend");
    a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
    a.bcast = (decltype(a.bcast))dlsym(h, "ncclBroadcast");
    a.err = (decltype(a.err))dlsym(h, "ncclGetErrorString");
    a.ok = a.group_start && a.group_end && a.send && a.recv && a.bcast && a.err;
    return a;
  }();
  return api;
}

struct SpLayout {
  int64_t n_local, sink_rows, halo_rows;
  int64_t k_row_elems, v_row_elems;  // elements per exchanged row (v: 0 when v aliases k)
  size_t esz;
  size_t sink_k_off, sink_v_off, halo_k_off, halo_v_off, total;
};

loza_status_t sp_layout(const loza_attn_args_t* a, loza_pattern_t pat, SpLayout* L) {
  if (!a) return fail(LOZA_ERR_INVALID, "args is NULL");
  if (pat.sink_blocks < 0 || pat.local_blocks < 1 || pat.block_size < 1) return fail(LOZA_ERR_INVALID, "bad pattern");
  if (a->batch < 0 || a->n_q < 0) return fail(LOZA_ERR_SHAPE, "negative dimension");
  const int64_t b = pat.block_size;
  L->n_local = a->n_q;
  if (a->n_kv != a->n_q) return fail(LOZA_ERR_SHAPE, "seqpar: k/v must hold exactly the shard's rows (n_kv == n_q)");
  if (L->n_local % b) return fail(LOZA_ERR_SHAPE, "seqpar: shard length must be a multiple of b");
  L->sink_rows = (int64_t)pat.sink_blocks * b;
  L->halo_rows = (int64_t)(pat.local_blocks - 1) * b;
  if (L->n_local < L->sink_rows || L->n_local < L->halo_rows)
    return fail(LOZA_ERR_SHAPE, "seqpar: shard shorter than the sink or halo (need >= max(s, l-1)*b rows)");
  const bool alias = a->v == a->k;
  L->esz = a->in_dtype == LOZA_BF16 ? 2 : 4;
  L->k_row_elems = a->d_qk;
  L->v_row_elems = alias ? 0 : a->d_v;
  const size_t B = (size_t)a->batch;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  L->sink_k_off = take(B * L->sink_rows * L->k_row_elems * L->esz);
  L->sink_v_off = take(B * L->sink_rows * L->v_row_elems * L->esz);
  L->halo_k_off = take(B * L->halo_rows * L->k_row_elems * L->esz);
  L->halo_v_off = take(B * L->halo_rows * L->v_row_elems * L->esz);
  L->total = off;
  return LOZA_OK;
}

loza_status_t sp_validate(const loza_attn_args_t* a, loza_pattern_t pat, int32_t rank, int32_t world, SpLayout* L) {
  if (world < 1 || rank < 0 || rank >= world) return fail(LOZA_ERR_INVALID, "bad rank/world");
  loza_status_t rc = sp_layout(a, pat, L);
  if (rc != LOZA_OK) return rc;
  if (a->q_start != (int64_t)rank * L->n_local) return fail(LOZA_ERR_SHAPE, "seqpar: q_start must be rank * n_local");
  if (a->k_stride_tok != a->d_qk || (a->v != a->k && a->v_stride_tok != a->d_v))
    return fail(LOZA_ERR_UNSUPPORTED, "seqpar: k/v rows must be contiguous (stride_tok == d)");
  return LOZA_OK;
}

// The exchange plan of `rank` (loza.h: loza_seqpar_plan), in issue order: group 1 = the sink broadcasts,
// group 2 = the halo sends / receives. Every rank lists the same broadcasts, and rank r's SEND to r+1
// matches rank r+1's RECV from r entry for entry.
int sp_plan(const loza_attn_args_t* a, const SpLayout& L, int32_t rank, int32_t world, loza_xfer_t* out, int max_out) {
  int n = 0;
  auto put = [&](loza_xfer_t x) { if (n < max_out) out[n] = x; ++n; };
  if (world <= 1) return 0;
  const bool alias = a->v == a->k;
  const int ntens = alias ? 1 : 2;
  for (int32_t bi = 0; bi < a->batch; ++bi)
    for (int t = 0; t < ntens && L.sink_rows > 0; ++t) {
      const int64_t re = t ? L.v_row_elems : L.k_row_elems;
      const size_t base = t ? L.sink_v_off : L.sink_k_off;
      put(loza_xfer_t{LOZA_XFER_BCAST, 0, bi, t, 0, L.sink_rows, re,
                      rank == 0 ? -1 : (int64_t)(base + (size_t)bi * L.sink_rows * re * L.esz)});
    }
  if (L.halo_rows == 0) return n;
  const int64_t last = L.n_local - L.halo_rows;
  for (int32_t bi = 0; bi < a->batch; ++bi)
    for (int t = 0; t < ntens; ++t) {
      const int64_t re = t ? L.v_row_elems : L.k_row_elems;
      const size_t base = t ? L.halo_v_off : L.halo_k_off;
      if (rank + 1 < world) put(loza_xfer_t{LOZA_XFER_SEND, rank + 1, bi, t, last, L.halo_rows, re, -1});
      if (rank > 0)
        put(loza_xfer_t{LOZA_XFER_RECV, rank - 1, bi, t, last, L.halo_rows, re,
                        (int64_t)(base + (size_t)bi * L.halo_rows * re * L.esz)});
    }
  return n;
}

// Segmented KV view of `rank` once sink/halo rows sit in ws: segment i has k/v rows at ws + k_off[i] /
// ws + v_off[i] (-1: the shard's own k/v).
int sp_segments(const loza_attn_args_t* a, const SpLayout& L, int32_t rank, KvSeg* seg, int64_t* k_off,
                int64_t* v_off) {
  const int64_t q0 = a->q_start;
  const bool alias = a->v == a->k;
  int n = 0;
  const int64_t kr = L.k_row_elems, vr = alias ? kr : L.v_row_elems;
  if (rank > 0 && L.sink_rows > 0) {
    k_off[n] = (int64_t)L.sink_k_off;
    v_off[n] = alias ? k_off[n] : (int64_t)L.sink_v_off;
    seg[n++] = KvSeg{0, L.sink_rows, nullptr, nullptr, L.sink_rows * kr, kr, L.sink_rows * vr, vr};
  }
  if (rank > 0 && L.halo_rows > 0) {
    // halo = positions [q0 - halo_rows, q0); clipped where it overlaps the sink segment
    int64_t begin = q0 - L.halo_rows, skip = 0;
    if (n > 0 && begin < L.sink_rows) { skip = L.sink_rows - begin; begin = L.sink_rows; }
    if (begin < q0) {
      k_off[n] = (int64_t)(L.halo_k_off + (size_t)skip * kr * L.esz);
      v_off[n] = alias ? k_off[n] : (int64_t)(L.halo_v_off + (size_t)skip * vr * L.esz);
      seg[n++] = KvSeg{begin, q0, nullptr, nullptr, L.halo_rows * kr, kr, L.halo_rows * vr, vr};
    }
  }
  k_off[n] = v_off[n] = -1;
  seg[n++] = KvSeg{q0, q0 + L.n_local, a->k, a->v, a->k_stride_b, a->k_stride_tok, a->v_stride_b, a->v_stride_tok};
  return n;
}

void sp_view(const loza_attn_args_t* a, const SpLayout& L, int32_t rank, char* ws, KvView* kv) {
  int64_t k_off[3], v_off[3];
  kv->nseg = sp_segments(a, L, rank, kv->seg, k_off, v_off);
  for (int i = 0; i < kv->nseg; ++i)
    if (k_off[i] >= 0) {
      kv->seg[i].k = ws + k_off[i];
      kv->seg[i].v = ws + v_off[i];
    }
}

// Per (host thread, device): the communication stream and two events of the split launch.
struct CommCtx {
  cudaStream_t comm = nullptr;
  cudaEvent_t fork = nullptr, halo = nullptr;
};
loza_status_t comm_ctx(CommCtx** out) {
  static thread_local CommCtx ctx[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return fail(LOZA_ERR_UNSUPPORTED, "device index >= 64");
  CommCtx& c = ctx[dev];
  if (!c.comm) {
    e = cudaStreamCreateWithFlags(&c.comm, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.halo, cudaEventDisableTiming);
    if (e != cudaSuccess) { c.comm = nullptr; return cuda_status(e, "seqpar comm stream"); }
  }
  *out = &c;
  return LOZA_OK;
}

enum class Backend { kNccl, kVirtual, kLoopback };
struct PeerBufs { const void *rank0_k, *rank0_v, *prev_k, *prev_v; };

const char* row_ptr(const void* base, const loza_attn_args_t* a, const loza_xfer_t& x, size_t esz) {
  const int64_t sb = x.tensor ? a->v_stride_b : a->k_stride_b;
  return reinterpret_cast<const char*>(base) + ((size_t)x.batch * sb + (size_t)x.src_row * x.row_elems) * esz;
}

// Issue one group of the plan (group 1: BCAST entries on st; group 2: SEND/RECV entries on st).
loza_status_t run_group(int group, Backend be, const loza_xfer_t* plan, int n, const loza_attn_args_t* a,
                        const SpLayout& L, int32_t rank, char* ws, void* comm, const PeerBufs& pb, cudaStream_t st) {
  const bool nccl_be = be != Backend::kVirtual;
  const NcclApi* api = nullptr;
  ncclDataType_t dt = a->in_dtype == LOZA_BF16 ? ncclBfloat16 : ncclFloat32;
  ncclComm_t c = (ncclComm_t)comm;
  ncclResult_t r = ncclSuccess;
  if (nccl_be) {
    api = &nccl();
    if (!api->ok) return fail(LOZA_ERR_NCCL, "libnccl.so.2 not loadable");
    r = api->group_start();
  }
  for (int i = 0; i < n && r == ncclSuccess; ++i) {
    const loza_xfer_t& x = plan[i];
    const bool in_group = group == 1 ? x.op == LOZA_XFER_BCAST : x.op != LOZA_XFER_BCAST;
    if (!in_group) continue;
    const size_t count = (size_t)x.rows * x.row_elems;
    const void* own = x.tensor ? a->v : a->k;
    char* dst = x.ws_offset >= 0 ? ws + x.ws_offset : nullptr;
    if (be == Backend::kNccl) {
      if (x.op == LOZA_XFER_BCAST) {
        const char* src = row_ptr(own, a, x, L.esz);  // read on the root only
        r = api->bcast(src, dst ? dst : const_cast<char*>(src), count, dt, x.peer, c, st);
      } else if (x.op == LOZA_XFER_SEND) {
        r = api->send(row_ptr(own, a, x, L.esz), count, dt, x.peer, c, st);
      } else {
        r = api->recv(dst, count, dt, x.peer, c, st);
      }
    } else {
      // virtual ranks: the sender's rows are another shard on this GPU
      const void* peer_base = x.op == LOZA_XFER_BCAST ? (x.tensor ? pb.rank0_v : pb.rank0_k)
                                                      : (x.tensor ? pb.prev_v : pb.prev_k);
      if (x.op == LOZA_XFER_SEND || !dst) continue;  // matched by the receiving virtual rank / root keeps rows
      if (!peer_base) return fail(LOZA_ERR_INVALID, "seqpar test hook: missing rank-0 / previous shard buffer");
      const char* src = row_ptr(peer_base, a, x, L.esz);
      if (be == Backend::kVirtual) {
        cudaError_t e = cudaMemcpyAsync(dst, src, count * L.esz, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_status(e, "seqpar local copy");
      } else if (x.op == LOZA_XFER_BCAST) {  // loopback: one-rank communicator, root 0 = this process
        r = api->bcast(src, dst, count, dt, 0, c, st);
      } else {
        r = api->send(src, count, dt, 0, c, st);
        if (r == ncclSuccess) r = api->recv(dst, count, dt, 0, c, st);
      }
    }
  }
  if (nccl_be) {
    ncclResult_t r2 = api->group_end();
    if (r != ncclSuccess) return fail(LOZA_ERR_NCCL, "nccl (group %d): %s", group, api->err(r));
    if (r2 != ncclSuccess) return fail(LOZA_ERR_NCCL, "nccl group %d end: %s", group, api->err(r2));
  }
  (void)rank;
  return LOZA_OK;
}

// A query sub-range [t0, t0 + nt) of the shard's problem (pointers and q_start shifted, lse head stride kept).
AttnProblem sub_problem(const AttnProblem& p, const loza_attn_args_t* a, int64_t t0, int64_t nt) {
  AttnProblem s = p;
  const size_t iesz = a->in_dtype == LOZA_BF16 ? 2 : 4, oesz = a->out_dtype == LOZA_BF16 ? 2 : 4;
  s.q = reinterpret_cast<const char*>(p.q) + (size_t)t0 * p.q_st * iesz;
  s.o = reinterpret_cast<char*>(p.o) + (size_t)t0 * p.o_st * oesz;
  if (p.lse) s.lse = p.lse + t0;
  s.n_q = (int32_t)nt;
  s.q_start = p.q_start + t0;
  return s;
}

// Exchange (per backend) + the split SSA launch of the shard.
loza_status_t sp_run(Backend be, const loza_attn_args_t* a, loza_pattern_t pat, void* comm, int32_t rank,
                     int32_t world, const PeerBufs& pb, void* ws, size_t ws_bytes, cudaStream_t st) {
  SpLayout L;
  loza_status_t rc = sp_validate(a, pat, rank, world, &L);
  if (rc != LOZA_OK) return rc;
  // the shard's own problem: queries [q_start, q_start+n_local) against keys [0, q_start+n_local)
  loza_attn_args_t g = *a;
  g.n_kv = a->q_start + L.n_local;
  AttnProblem p;
  rc = make_problem(&g, true, pat, nullptr, &p);
  if (rc != LOZA_OK) return rc;
  const bool exchange = world > 1 || (be != Backend::kNccl && rank > 0);
  if (!exchange) return run_attention(&g, p, nullptr, 0, st);
  if (be == Backend::kNccl && !comm) return fail(LOZA_ERR_INVALID, "seqpar: NULL communicator with world > 1");
  if (L.total > 0 && (!ws || ws_bytes < L.total))
    return fail(LOZA_ERR_INVALID, "seqpar workspace too small (%zu < %zu)", ws_bytes, L.total);
  char* w = reinterpret_cast<char*>(ws);
  loza_xfer_t plan[64];
  const int nplan = sp_plan(a, L, rank, world, plan, 64);
  if (nplan > 64) return fail(LOZA_ERR_UNSUPPORTED, "seqpar: more than 64 transfers (batch too large)");
  CommCtx* cc = nullptr;
  if ((rc = comm_ctx(&cc)) != LOZA_OK) return rc;
  cudaError_t e = cudaEventRecord(cc->fork, st);  // inputs produced on st are ready for the halo group
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cc->comm, cc->fork, 0);
  if (e != cudaSuccess) return cuda_status(e, "seqpar fork");
  // group 1 (sink broadcast) on st: every query block of the shard needs it
  if ((rc = run_group(1, be, plan, nplan, a, L, rank, w, comm, pb, st)) != LOZA_OK) return rc;
  // group 2 (halo) on the comm stream, issued before the interior launch so its kernel gets SMs first
  if ((rc = run_group(2, be, plan, nplan, a, L, rank, w, comm, pb, cc->comm)) != LOZA_OK) return rc;
  if ((e = cudaEventRecord(cc->halo, cc->comm)) != cudaSuccess) return cuda_status(e, "seqpar halo event");
  sp_view(a, L, rank, w, &p.kv);
  const int64_t halo_q = rank > 0 ? (L.halo_rows < L.n_local ? L.halo_rows : L.n_local) : 0;
  if (halo_q < L.n_local) {  // interior query blocks: [sink | shard] only
    const AttnProblem pi = halo_q ? sub_problem(p, a, halo_q, L.n_local - halo_q) : p;
    if ((rc = run_attention(&g, pi, nullptr, 0, st)) != LOZA_OK) return rc;
  }
  // the first l-1 blocks read the halo; st also joins the comm stream here (rank 0 included)
  if ((e = cudaStreamWaitEvent(st, cc->halo, 0)) != cudaSuccess) return cuda_status(e, "seqpar join");
  if (halo_q > 0) return run_attention(&g, sub_problem(p, a, 0, halo_q), nullptr, 0, st);
  return LOZA_OK;
}

}  // namespace
}  // namespace loza

using namespace loza;

extern "C" size_t loza_seqpar_ws_bytes(const loza_attn_args_t* a, loza_pattern_t pat) {
  SpLayout L;
  if (sp_layout(a, pat, &L) != LOZA_OK) return 0;
  return L.total;
}

extern "C" int32_t loza_seqpar_plan(const loza_attn_args_t* a, loza_pattern_t pat, int32_t rank, int32_t world,
                                    loza_xfer_t* out, int32_t max_out) {
  SpLayout L;
  loza_status_t rc = sp_validate(a, pat, rank, world, &L);
  if (rc != LOZA_OK) return -(int32_t)rc;
  if (max_out > 0 && !out) return -(int32_t)fail(LOZA_ERR_INVALID, "out is NULL");
  return sp_plan(a, L, rank, world, out, max_out < 0 ? 0 : max_out);
}

extern "C" int32_t loza_seqpar_segments(const loza_attn_args_t* a, loza_pattern_t pat, int32_t rank, int32_t world,
                                        int64_t* seg_out) {
  SpLayout L;
  loza_status_t rc = sp_validate(a, pat, rank, world, &L);
  if (rc != LOZA_OK) return -(int32_t)rc;
  if (!seg_out) return -(int32_t)fail(LOZA_ERR_INVALID, "seg_out is NULL");
  KvSeg seg[3];
  int64_t k_off[3], v_off[3];
  const int n = sp_segments(a, L, rank, seg, k_off, v_off);
  const int64_t esz = (int64_t)L.esz;
  for (int i = 0; i < n; ++i) {
    int64_t* o = seg_out + 6 * i;
    o[0] = seg[i].pos_begin;
    o[1] = seg[i].pos_end;
    o[2] = k_off[i];
    o[3] = v_off[i];
    o[4] = seg[i].k_sb * esz;
    o[5] = seg[i].v_sb * esz;
  }
  return n;
}

extern "C" loza_status_t ssa_seqpar_prefill(const loza_attn_args_t* a, loza_pattern_t pat, loza_nccl_comm_t comm,
                                            int32_t rank, int32_t world, void* ws, size_t ws_bytes,
                                            loza_stream_t stream) {
  return sp_run(Backend::kNccl, a, pat, comm, rank, world, PeerBufs{}, ws, ws_bytes, (cudaStream_t)stream);
}

// Test hook ("virtual ranks"): the plan's transfers as device-to-device copies from the
// other shards' buffers on this GPU, then the same split launch.
extern "C" loza_status_t loza_seqpar_prefill_local(const loza_attn_args_t* a, loza_pattern_t pat, int32_t rank,
                                                   int32_t world, const void* rank0_k, const void* rank0_v,
                                                   const void* prev_k, const void* prev_v, void* ws,
                                                   size_t ws_bytes, loza_stream_t stream) {
  return sp_run(Backend::kVirtual, a, pat, nullptr, rank, world, PeerBufs{rank0_k, rank0_v, prev_k, prev_v}, ws,
                ws_bytes, (cudaStream_t)stream);
}

// Test hook ("NCCL loopback"): the plan's transfers through NCCL on a one-rank communicator.
extern "C" loza_status_t loza_seqpar_prefill_loopback(const loza_attn_args_t* a, loza_pattern_t pat,
                                                      loza_nccl_comm_t comm, int32_t rank, int32_t world,
                                                      const void* rank0_k, const void* rank0_v, const void* prev_k,
                                                      const void* prev_v, void* ws, size_t ws_bytes,
                                                      loza_stream_t stream) {
  if (!comm) return fail(LOZA_ERR_INVALID, "loopback: NULL communicator");
  return sp_run(Backend::kLoopback, a, pat, comm, rank, world, PeerBufs{rank0_k, rank0_v, prev_k, prev_v}, ws,
                ws_bytes, (cudaStream_t)stream);
}
