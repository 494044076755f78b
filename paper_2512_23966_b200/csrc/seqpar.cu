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
  const size_t B = (size_t)(a->batch > 0 ? a->batch : 0);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  L->sink_k_off = take(B * L->sink_rows * L->k_row_elems * L->esz);
  L->sink_v_off = take(B * L->sink_rows * L->v_row_elems * L->esz);
  L->halo_k_off = take(B * L->halo_rows * L->k_row_elems * L->esz);
  L->halo_v_off = take(B * L->halo_rows * L->v_row_elems * L->esz);
  L->total = off;
  return LOZA_OK;
}

// Segmented KV view for the shard of `rank` once sink/halo rows sit in ws.
void sp_view(const loza_attn_args_t* a, const SpLayout& L, int32_t rank, char* ws, KvView* kv) {
  const int64_t q0 = a->q_start;
  const bool alias = a->v == a->k;
  int n = 0;
  if (rank > 0 && L.sink_rows > 0) {
    const char* sk = ws + L.sink_k_off;
    const char* sv = alias ? sk : ws + L.sink_v_off;
    const int64_t kr = L.k_row_elems, vr = alias ? kr : L.v_row_elems;
    kv->seg[n++] = KvSeg{0, L.sink_rows, sk, sv, L.sink_rows * kr, kr, L.sink_rows * vr, vr};
  }
  if (rank > 0 && L.halo_rows > 0) {
    // halo = positions [q0 - halo_rows, q0); clip where it overlaps the sink segment
    int64_t begin = q0 - L.halo_rows, skip = 0;
    if (n > 0 && begin < L.sink_rows) { skip = L.sink_rows - begin; begin = L.sink_rows; }
    const int64_t kr = L.k_row_elems, vr = alias ? kr : L.v_row_elems;
    const char* hk = ws + L.halo_k_off + (size_t)skip * kr * L.esz;
    const char* hv = alias ? hk : ws + L.halo_v_off + (size_t)skip * vr * L.esz;
    if (begin < q0) kv->seg[n++] = KvSeg{begin, q0, hk, hv, L.halo_rows * kr, kr, L.halo_rows * vr, vr};
  }
  kv->seg[n++] = KvSeg{q0, q0 + L.n_local, a->k, a->v, a->k_stride_b, a->k_stride_tok, a->v_stride_b,
                       a->v_stride_tok};
  kv->nseg = n;
}

loza_status_t sp_compute(const loza_attn_args_t* a, loza_pattern_t pat, const SpLayout& L, int32_t rank, void* ws,
                         cudaStream_t st) {
  // the shard's own problem: queries [q_start, q_start+n_local) against keys [0, q_start+n_local)
  loza_attn_args_t g = *a;
  g.n_kv = a->q_start + L.n_local;
  AttnProblem p;
  loza_status_t rc = make_problem(&g, true, pat, nullptr, &p);
  if (rc != LOZA_OK) return rc;
  sp_view(a, L, rank, reinterpret_cast<char*>(ws), &p.kv);
  return run_attention(&g, p, nullptr, 0, st);
}

loza_status_t check_rows_contiguous(const loza_attn_args_t* a) {
  if (a->k_stride_tok != a->d_qk || (a->v != a->k && a->v_stride_tok != a->d_v))
    return fail(LOZA_ERR_UNSUPPORTED, "seqpar: k/v rows must be contiguous (stride_tok == d)");
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

extern "C" loza_status_t ssa_seqpar_prefill(const loza_attn_args_t* a, loza_pattern_t pat, loza_nccl_comm_t comm,
                                            int32_t rank, int32_t world, void* ws, size_t ws_bytes,
                                            loza_stream_t stream) {
  if (world < 1 || rank < 0 || rank >= world) return fail(LOZA_ERR_INVALID, "bad rank/world");
  SpLayout L;
  loza_status_t rc = sp_layout(a, pat, &L);
  if (rc != LOZA_OK) return rc;
  if (a->q_start != (int64_t)rank * L.n_local) return fail(LOZA_ERR_SHAPE, "seqpar: q_start must be rank * n_local");
  if ((rc = check_rows_contiguous(a)) != LOZA_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (world > 1) {
    if (!comm) return fail(LOZA_ERR_INVALID, "seqpar: NULL communicator with world > 1");
    if (!ws || ws_bytes < L.total) return fail(LOZA_ERR_INVALID, "seqpar workspace too small (%zu < %zu)", ws_bytes, L.total);
    const NcclApi& api = nccl();
    if (!api.ok) return fail(LOZA_ERR_NCCL, "libnccl.so.2 not loadable");
    const ncclDataType_t dt = a->in_dtype == LOZA_BF16 ? ncclBfloat16 : ncclFloat32;
    ncclComm_t c = (ncclComm_t)comm;
    char* w = reinterpret_cast<char*>(ws);
    const bool alias = a->v == a->k;
    ncclResult_t r = api.group_start();
    for (int32_t bi = 0; bi < a->batch && r == ncclSuccess; ++bi) {
      const char* kb = reinterpret_cast<const char*>(a->k) + (size_t)bi * a->k_stride_b * L.esz;
      const char* vb = reinterpret_cast<const char*>(a->v) + (size_t)bi * a->v_stride_b * L.esz;
      if (L.sink_rows > 0) {
        const size_t nk = (size_t)L.sink_rows * L.k_row_elems;
        r = api.bcast(kb, w + L.sink_k_off + bi * nk * L.esz, nk, dt, 0, c, st);
        if (r == ncclSuccess && !alias) {
          const size_t nv = (size_t)L.sink_rows * L.v_row_elems;
          r = api.bcast(vb, w + L.sink_v_off + bi * nv * L.esz, nv, dt, 0, c, st);
        }
      }
      if (L.halo_rows > 0 && r == ncclSuccess) {
        const size_t nk = (size_t)L.halo_rows * L.k_row_elems;
        const size_t nv = (size_t)L.halo_rows * L.v_row_elems;
        const int64_t last = L.n_local - L.halo_rows;
        if (rank + 1 < world) {
          r = api.send(kb + (size_t)last * L.k_row_elems * L.esz, nk, dt, rank + 1, c, st);
          if (r == ncclSuccess && !alias) r = api.send(vb + (size_t)last * L.v_row_elems * L.esz, nv, dt, rank + 1, c, st);
        }
        if (rank > 0 && r == ncclSuccess) {
          r = api.recv(w + L.halo_k_off + bi * nk * L.esz, nk, dt, rank - 1, c, st);
          if (r == ncclSuccess && !alias) r = api.recv(w + L.halo_v_off + bi * nv * L.esz, nv, dt, rank - 1, c, st);
        }
      }
    }
    ncclResult_t r2 = api.group_end();
    if (r != ncclSuccess) return fail(LOZA_ERR_NCCL, "nccl: %s", api.err(r));
    if (r2 != ncclSuccess) return fail(LOZA_ERR_NCCL, "nccl group end: %s", api.err(r2));
  }
  return sp_compute(a, pat, L, rank, ws, st);
}

// Test hook ("virtual ranks"): the same exchange done with
// device-to-device copies from the other shards' buffers on this GPU
// (rank0_k/v = rank 0's shard base, prev_k/v = rank-1's shard base), then the
// same compute step. Lets the partition and halo logic be checked bitwise
// against the single-GPU prefill without a multi-GPU box.
extern "C" loza_status_t loza_seqpar_prefill_local(const loza_attn_args_t* a, loza_pattern_t pat, int32_t rank,
                                                   int32_t world, const void* rank0_k, const void* rank0_v,
                                                   const void* prev_k, const void* prev_v, void* ws,
                                                   size_t ws_bytes, loza_stream_t stream) {
  if (world < 1 || rank < 0 || rank >= world) return fail(LOZA_ERR_INVALID, "bad rank/world");
  SpLayout L;
  loza_status_t rc = sp_layout(a, pat, &L);
  if (rc != LOZA_OK) return rc;
  if (a->q_start != (int64_t)rank * L.n_local) return fail(LOZA_ERR_SHAPE, "seqpar: q_start must be rank * n_local");
  if ((rc = check_rows_contiguous(a)) != LOZA_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (rank > 0) {
    if (!ws || ws_bytes < L.total) return fail(LOZA_ERR_INVALID, "seqpar workspace too small");
    char* w = reinterpret_cast<char*>(ws);
    const bool alias = a->v == a->k;
    for (int32_t bi = 0; bi < a->batch; ++bi) {
      const size_t boff_k = (size_t)bi * a->k_stride_b * L.esz, boff_v = (size_t)bi * a->v_stride_b * L.esz;
      cudaError_t e = cudaSuccess;
      if (L.sink_rows > 0) {
        const size_t nk = (size_t)L.sink_rows * L.k_row_elems * L.esz;
        e = cudaMemcpyAsync(w + L.sink_k_off + bi * nk, (const char*)rank0_k + boff_k, nk, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && !alias) {
          const size_t nv = (size_t)L.sink_rows * L.v_row_elems * L.esz;
          e = cudaMemcpyAsync(w + L.sink_v_off + bi * nv, (const char*)rank0_v + boff_v, nv, cudaMemcpyDeviceToDevice, st);
        }
      }
      if (L.halo_rows > 0 && e == cudaSuccess) {
        const int64_t last = L.n_local - L.halo_rows;
        const size_t nk = (size_t)L.halo_rows * L.k_row_elems * L.esz;
        e = cudaMemcpyAsync(w + L.halo_k_off + bi * nk, (const char*)prev_k + boff_k + last * L.k_row_elems * L.esz, nk,
                            cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && !alias) {
          const size_t nv = (size_t)L.halo_rows * L.v_row_elems * L.esz;
          e = cudaMemcpyAsync(w + L.halo_v_off + bi * nv, (const char*)prev_v + boff_v + last * L.v_row_elems * L.esz,
                              nv, cudaMemcpyDeviceToDevice, st);
        }
      }
      if (e != cudaSuccess) return cuda_status(e, "seqpar local copy");
    }
  }
  return sp_compute(a, pat, L, rank, ws, st);
}
