// C-ABI entry points of libloza.so: host-side validation, dispatch, errors.
// See include/loza.h for the contract of each call.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>

#include "internal.h"

namespace loza {

static thread_local char g_last_error[512] = {0};
static std::atomic<uint64_t> g_launches{0};

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static std::atomic<int> g_knobs[kNumKnobs];
int knob(KnobFamily f) { return g_knobs[f].load(std::memory_order_relaxed); }

int device_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}

loza_status_t fail(loza_status_t st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return st;
}

loza_status_t cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return LOZA_OK;
  return fail(LOZA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Validate the common part of an attention call and fill an AttnProblem.
loza_status_t make_problem(const loza_attn_args_t* a, bool sparse, loza_pattern_t pat, const int32_t* seq_lens,
                           AttnProblem* p) {
  if (!a) return fail(LOZA_ERR_INVALID, "args is NULL");
  if (!isfinite(a->softmax_scale)) return fail(LOZA_ERR_INVALID, "softmax_scale is not finite");
  if (a->causal != 0 && a->causal != 1) return fail(LOZA_ERR_INVALID, "causal must be 0 or 1");
  if (sparse) {
    if (pat.sink_blocks < 0 || pat.local_blocks < 1 || pat.block_size < 1)
      return fail(LOZA_ERR_INVALID, "pattern needs s >= 0, l >= 1, b >= 1 (got %d, %d, %d)", pat.sink_blocks,
                  pat.local_blocks, pat.block_size);
    if (!a->causal) return fail(LOZA_ERR_UNSUPPORTED, "SSA is causal only (DESIGN R9)");
  }
  if (a->batch < 0 || a->n_q < 0 || a->heads < 1 || a->d_qk < 1 || a->d_v < 1 || a->n_kv < 0 || a->q_start < 0)
    return fail(LOZA_ERR_SHAPE, "negative or zero dimension");
  if ((a->in_dtype != LOZA_F32 && a->in_dtype != LOZA_BF16) || (a->out_dtype != LOZA_F32 && a->out_dtype != LOZA_BF16))
    return fail(LOZA_ERR_INVALID, "unknown dtype");
  if (seq_lens) {
    if (a->n_q != 1) return fail(LOZA_ERR_SHAPE, "decode needs n_q == 1");
    if (a->n_kv < 1) return fail(LOZA_ERR_SHAPE, "decode needs n_kv (cache capacity) >= 1");
  } else {
    if (a->causal && a->n_kv < a->q_start + a->n_q)
      return fail(LOZA_ERR_SHAPE, "n_kv (%lld) < q_start + n_q (%lld)", (long long)a->n_kv,
                  (long long)(a->q_start + a->n_q));
    if (sparse && a->q_start % pat.block_size != 0)
      return fail(LOZA_ERR_SHAPE, "q_start must be a multiple of b");
  }
  const bool empty = (int64_t)a->batch * a->n_q * a->heads == 0;
  if (!empty && (!a->q || !a->k || !a->v || !a->o)) return fail(LOZA_ERR_INVALID, "NULL tensor pointer");
  memset(p, 0, sizeof(*p));
  p->batch = a->batch; p->n_q = a->n_q; p->heads = a->heads; p->d_qk = a->d_qk; p->d_v = a->d_v;
  p->n_kv = a->n_kv; p->q_start = a->q_start;
  p->in_bf16 = a->in_dtype == LOZA_BF16; p->out_bf16 = a->out_dtype == LOZA_BF16;
  p->scale = a->softmax_scale; p->causal = a->causal; p->sparse = sparse ? 1 : 0;
  p->s = sparse ? pat.sink_blocks : 0; p->l = sparse ? pat.local_blocks : 1; p->b = sparse ? pat.block_size : 1;
  p->q = a->q; p->q_sb = a->q_stride_b; p->q_st = a->q_stride_tok; p->q_sh = a->q_stride_head;
  p->o = a->o; p->o_sb = a->o_stride_b; p->o_st = a->o_stride_tok; p->o_sh = a->o_stride_head;
  p->lse = a->lse; p->lse_sh = a->n_q; p->seq_lens = seq_lens;
  p->kv.nseg = 1;
  p->kv.seg[0] = KvSeg{0, a->n_kv, a->k, a->v, a->k_stride_b, a->k_stride_tok, a->v_stride_b, a->v_stride_tok};
  return LOZA_OK;
}

// Route a validated problem to its kernel family (no fallback).
enum class Path { kSimt, kTc };
loza_status_t choose_path(const loza_attn_args_t* a, const AttnProblem& p, Path* path) {
  if (a->in_dtype == LOZA_F32) {
    if (a->d_qk > 576 || a->d_v > 512)
      return fail(LOZA_ERR_UNSUPPORTED, "fp32 path supports d_qk <= 576, d_v <= 512");
    *path = Path::kSimt;
    return LOZA_OK;
  }
  if (a->d_qk != 576 || a->d_v != 512)
    return fail(LOZA_ERR_UNSUPPORTED, "bf16 path supports the absorbed MLA shape (576, 512) only");
  if (p.sparse && p.b % 128 != 0) return fail(LOZA_ERR_UNSUPPORTED, "bf16 SSA path needs b %% 128 == 0");
  const int64_t esz = 2;
  if (!aligned16(a->q) || !aligned16(a->k) || !aligned16(a->v) || !aligned16(a->o))
    return fail(LOZA_ERR_SHAPE, "bf16 path needs 16-byte aligned base pointers");
  if ((a->k_stride_tok * esz) % 16 || (a->k_stride_b * esz) % 16 || (a->v_stride_tok * esz) % 16 ||
      (a->v_stride_b * esz) % 16 || (a->q_stride_b * esz) % 16 || (a->q_stride_tok * esz) % 16 ||
      (a->q_stride_head * esz) % 16)
    return fail(LOZA_ERR_SHAPE, "bf16 path needs 16-byte aligned strides");
  if (a->out_dtype == LOZA_BF16 &&
      ((a->o_stride_b * esz) % 16 || (a->o_stride_tok * esz) % 16 || (a->o_stride_head * esz) % 16))
    return fail(LOZA_ERR_SHAPE, "bf16 output needs 16-byte aligned strides (16-byte / TMA stores)");
  if (!p.seq_lens) {
    if (a->q_stride_head != a->d_qk || a->q_stride_tok != (int64_t)a->heads * a->d_qk)
      return fail(LOZA_ERR_UNSUPPORTED, "bf16 prefill needs head-contiguous q rows");
    if (a->o_stride_head != a->d_v || a->o_stride_tok != (int64_t)a->heads * a->d_v)
      return fail(LOZA_ERR_UNSUPPORTED, "bf16 prefill needs head-contiguous o rows");
    if (p.sparse && ((int64_t)a->heads * p.b) % 128 != 0)
      return fail(LOZA_ERR_UNSUPPORTED, "bf16 prefill needs H*b %% 128 == 0");
    if (((int64_t)a->heads * a->n_q) % 128 != 0 && a->heads % 64 != 0)
      return fail(LOZA_ERR_UNSUPPORTED, "bf16 prefill needs H %% 64 == 0 or n_q*H %% 128 == 0");
  } else {
    // H < 64 (decode sharded by heads) runs on the key-split pair kernel, whose Q rows >= H are zero-filled
    if (a->heads > 64 || (a->heads != 64 && !decode_ks_eligible(p, device_sm_count())))
      return fail(LOZA_ERR_UNSUPPORTED, "bf16 decode supports H == 64, or H < 64 on the SSA pair kernel "
                                        "(2 * batch <= SMs, v aliasing k)");
    if (a->batch > 1024) return fail(LOZA_ERR_UNSUPPORTED, "bf16 decode supports batch <= 1024");
  }
  *path = Path::kTc;
  return LOZA_OK;
}

loza_status_t run_attention(const loza_attn_args_t* a, const AttnProblem& p, void* ws, size_t ws_bytes,
                            cudaStream_t st) {
  if ((int64_t)p.batch * p.n_q * p.heads == 0) return LOZA_OK;
  Path path;
  loza_status_t rc = choose_path(a, p, &path);
  if (rc != LOZA_OK) return rc;
  if (path == Path::kSimt) return cuda_status(launch_attn_simt(p, st), "attn_simt launch");
  if (p.seq_lens) {
    const size_t need = decode_tc_ws_bytes(p);
    if (need > 0 && (!ws || ws_bytes < need))
      return fail(LOZA_ERR_INVALID, "decode workspace too small (%zu < %zu)", ws_bytes, need);
    return cuda_status(launch_decode_tc(p, ws, ws_bytes, st), "decode_tc launch");
  }
  return cuda_status(launch_prefill_tc(p, st), "prefill_tc launch");
}

}  // namespace loza

using namespace loza;

extern "C" {

loza_status_t ssa_prefill(const loza_attn_args_t* args, loza_pattern_t pattern, loza_stream_t stream) {
  g_last_error[0] = 0;
  AttnProblem p;
  loza_status_t rc = make_problem(args, true, pattern, nullptr, &p);
  if (rc != LOZA_OK) return rc;
  return run_attention(args, p, nullptr, 0, (cudaStream_t)stream);
}

loza_status_t ssa_decode(const loza_attn_args_t* args, const int32_t* seq_lens_dev, loza_pattern_t pattern,
                         void* ws, size_t ws_bytes, loza_stream_t stream) {
  g_last_error[0] = 0;
  if (args && args->batch == 0) return LOZA_OK;  // nothing to decode (seq_lens may be NULL)
  if (!seq_lens_dev) return fail(LOZA_ERR_INVALID, "seq_lens_dev is NULL");
  AttnProblem p;
  loza_status_t rc = make_problem(args, true, pattern, seq_lens_dev, &p);
  if (rc != LOZA_OK) return rc;
  return run_attention(args, p, ws, ws_bytes, (cudaStream_t)stream);
}

loza_status_t full_attn_ref(const loza_attn_args_t* args, const int32_t* seq_lens_dev, void* ws, size_t ws_bytes,
                            loza_stream_t stream) {
  g_last_error[0] = 0;
  AttnProblem p;
  loza_pattern_t none = {0, 1, 1};
  loza_status_t rc = make_problem(args, false, none, seq_lens_dev, &p);
  if (rc != LOZA_OK) return rc;
  return run_attention(args, p, ws, ws_bytes, (cudaStream_t)stream);
}

loza_status_t loza_blend(const void* o_full, const void* o_sparse, const float* alpha_dev, void* o_hat,
                         const void* d_o_hat, double* d_alpha_dev, int64_t numel, loza_dtype_t dtype,
                         int32_t* status_dev, void* ws, size_t ws_bytes, loza_stream_t stream) {
  g_last_error[0] = 0;
  if (dtype != LOZA_F32 && dtype != LOZA_BF16) return fail(LOZA_ERR_INVALID, "unknown dtype");
  if (numel < 0 || numel % 8 != 0) return fail(LOZA_ERR_SHAPE, "numel must be a non-negative multiple of 8");
  if (!alpha_dev) return fail(LOZA_ERR_INVALID, "alpha_dev is NULL");
  if (numel == 0) return LOZA_OK;
  if (!o_full || !o_sparse) return fail(LOZA_ERR_INVALID, "NULL input");
  if ((d_o_hat == nullptr) != (d_alpha_dev == nullptr))
    return fail(LOZA_ERR_INVALID, "d_o_hat and d_alpha_dev must be both NULL or both set");
  if (!o_hat && !d_o_hat) return fail(LOZA_ERR_INVALID, "nothing to compute");
  if (!aligned16(o_full) || !aligned16(o_sparse) || (o_hat && !aligned16(o_hat)) || (d_o_hat && !aligned16(d_o_hat)))
    return fail(LOZA_ERR_SHAPE, "pointers must be 16-byte aligned");
  if (d_alpha_dev && (!ws || ws_bytes < blend_ws_bytes()))
    return fail(LOZA_ERR_INVALID, "blend workspace too small (%zu < %zu)", ws_bytes, blend_ws_bytes());
  return cuda_status(launch_blend(o_full, o_sparse, alpha_dev, o_hat, d_o_hat, d_alpha_dev, numel,
                                  dtype == LOZA_BF16, status_dev, ws, (cudaStream_t)stream),
                     "blend launch");
}

loza_status_t ssa_prefill_blend(const loza_attn_args_t* args, loza_pattern_t pattern, const void* o_full,
                                const float* alpha_dev, const void* d_o_hat, double* d_alpha_dev,
                                int32_t* status_dev, void* ws, size_t ws_bytes, loza_stream_t stream) {
  g_last_error[0] = 0;
  if (!alpha_dev) return fail(LOZA_ERR_INVALID, "alpha_dev is NULL");
  if (!o_full) return fail(LOZA_ERR_INVALID, "o_full is NULL");
  if ((d_o_hat == nullptr) != (d_alpha_dev == nullptr))
    return fail(LOZA_ERR_INVALID, "d_o_hat and d_alpha_dev must be both NULL or both set");
  AttnProblem p;
  loza_status_t rc = make_problem(args, true, pattern, nullptr, &p);
  if (rc != LOZA_OK) return rc;
  if (args->in_dtype != LOZA_BF16 || args->out_dtype != LOZA_BF16)
    return fail(LOZA_ERR_UNSUPPORTED, "ssa_prefill_blend: bf16 in and out only");
  Path path;
  rc = choose_path(args, p, &path);
  if (rc != LOZA_OK) return rc;
  if (path != Path::kTc) return fail(LOZA_ERR_UNSUPPORTED, "ssa_prefill_blend: tensor-core path only");
  if (!aligned16(o_full) || (d_o_hat && !aligned16(d_o_hat)))
    return fail(LOZA_ERR_SHAPE, "o_full / d_o_hat must be 16-byte aligned");
  if (d_alpha_dev && (!ws || ws_bytes < blend_ws_bytes() || (size_t)device_sm_count() * 8 > ws_bytes))
    return fail(LOZA_ERR_INVALID, "workspace too small (%zu < %zu)", ws_bytes, blend_ws_bytes());
  CalibArgs c{o_full, d_o_hat, alpha_dev, d_alpha_dev ? reinterpret_cast<double*>(ws) : nullptr, d_alpha_dev,
              status_dev};
  p.calib = &c;
  if ((int64_t)p.batch * p.n_q * p.heads == 0) return LOZA_OK;
  return cuda_status(launch_prefill_tc(p, (cudaStream_t)stream), "prefill_tc (calibration) launch");
}

loza_status_t attention_backward(const loza_attn_args_t* args, int32_t sparse, loza_pattern_t pattern,
                                 const void* d_o, float* d_q, float* d_k, float* d_v, void* ws, size_t ws_bytes,
                                 loza_stream_t stream) {
  g_last_error[0] = 0;
  if (sparse != 0 && sparse != 1) return fail(LOZA_ERR_INVALID, "sparse must be 0 or 1");
  AttnProblem p;
  loza_pattern_t none = {0, 1, 1};
  loza_status_t rc = make_problem(args, sparse != 0, sparse ? pattern : none, nullptr, &p);
  if (rc != LOZA_OK) return rc;
  if ((int64_t)p.batch * p.n_q == 0) {  // no query rows: every key gradient is zero (d_o, lse, d_q unused)
    if ((int64_t)p.batch * p.n_kv == 0) return LOZA_OK;
    if (!d_k || !d_v) return fail(LOZA_ERR_INVALID, "NULL gradient pointer");
    cudaError_t e = cudaMemsetAsync(d_k, 0, sizeof(float) * (size_t)p.batch * p.n_kv * args->d_qk, (cudaStream_t)stream);
    if (e == cudaSuccess)
      e = cudaMemsetAsync(d_v, 0, sizeof(float) * (size_t)p.batch * p.n_kv * args->d_v, (cudaStream_t)stream);
    return cuda_status(e, "backward (no query rows) memset");
  }
  if (!args->lse) return fail(LOZA_ERR_INVALID, "attention_backward needs the forward's lse");
  if (!d_o || !d_q || !d_k || !d_v) return fail(LOZA_ERR_INVALID, "NULL gradient pointer");
  if (args->d_qk > 576 || args->d_v > 512) return fail(LOZA_ERR_UNSUPPORTED, "d_qk <= 576 and d_v <= 512");
  if ((int64_t)p.batch * (p.n_q * (int64_t)p.heads + p.n_kv) == 0) return LOZA_OK;
  const size_t need = backward_ws_bytes(p);
  if (need > 0 && (!ws || ws_bytes < need)) return fail(LOZA_ERR_INVALID, "workspace too small (%zu < %zu)", ws_bytes, need);
  return cuda_status(launch_attn_backward(p, d_o, d_q, d_k, d_v, ws, (cudaStream_t)stream), "backward launch");
}

loza_status_t ssa_prefill_mha(const loza_attn_args_t* args, int64_t k_stride_head, int64_t v_stride_head,
                              int32_t sparse, loza_pattern_t pattern, loza_stream_t stream) {
  g_last_error[0] = 0;
  if (sparse != 0 && sparse != 1) return fail(LOZA_ERR_INVALID, "sparse must be 0 or 1");
  AttnProblem p;
  loza_pattern_t none = {0, 1, 1};
  loza_status_t rc = make_problem(args, sparse != 0, sparse ? pattern : none, nullptr, &p);
  if (rc != LOZA_OK) return rc;
  if (args->d_qk != 192 || args->d_v != 128)
    return fail(LOZA_ERR_UNSUPPORTED, "ssa_prefill_mha: per-head d_qk 192 (128 nope + 64 rope), d_v 128 only");
  if (args->in_dtype != LOZA_BF16) return fail(LOZA_ERR_UNSUPPORTED, "ssa_prefill_mha: bf16 inputs only");
  if (sparse && pattern.block_size % 128 != 0) return fail(LOZA_ERR_UNSUPPORTED, "ssa_prefill_mha needs b %% 128 == 0");
  if (!sparse && !args->causal && args->q_start != 0)
    return fail(LOZA_ERR_UNSUPPORTED, "bidirectional comparator needs q_start == 0");
  if ((int64_t)p.batch * p.n_q * p.heads == 0) return LOZA_OK;
  if (args->n_q > INT32_MAX / 2 || args->n_kv >= ((int64_t)1 << 31)) return fail(LOZA_ERR_SHAPE, "sizes too large");
  const int64_t esz = 2, oesz = args->out_dtype == LOZA_BF16 ? 2 : 4;
  if (!aligned16(args->q) || !aligned16(args->k) || !aligned16(args->v) || !aligned16(args->o))
    return fail(LOZA_ERR_SHAPE, "ssa_prefill_mha needs 16-byte aligned base pointers");
  const int64_t in_strides[] = {args->q_stride_b, args->q_stride_tok, args->q_stride_head, args->k_stride_b,
                                args->k_stride_tok, k_stride_head, args->v_stride_b, args->v_stride_tok, v_stride_head};
  for (int64_t s : in_strides)
    if (s < 0 || (s * esz) % 16) return fail(LOZA_ERR_SHAPE, "ssa_prefill_mha needs 16-byte aligned, non-negative strides");
  const int64_t o_strides[] = {args->o_stride_b, args->o_stride_tok, args->o_stride_head};
  for (int64_t s : o_strides)
    if (s < 0 || (s * oesz) % 16) return fail(LOZA_ERR_SHAPE, "ssa_prefill_mha needs 16-byte aligned output strides");
  return cuda_status(launch_prefill_mha(p, k_stride_head, v_stride_head, (cudaStream_t)stream), "prefill_mha launch");
}

loza_status_t ssa_ring_append(const void* rows, int64_t rows_stride_b, int64_t rows_stride_tok, int32_t m,
                              const int32_t* pos0_dev, loza_pattern_t pat, void* cache, int64_t cache_stride_b,
                              int64_t cache_stride_tok, int32_t batch, int32_t d, loza_dtype_t dtype,
                              loza_stream_t stream) {
  g_last_error[0] = 0;
  if (pat.sink_blocks < 0 || pat.local_blocks < 1 || pat.block_size < 1) return fail(LOZA_ERR_INVALID, "bad pattern");
  if (dtype != LOZA_F32 && dtype != LOZA_BF16) return fail(LOZA_ERR_INVALID, "unknown dtype");
  if (m < 0 || batch < 0 || d < 1) return fail(LOZA_ERR_SHAPE, "bad m / batch / d");
  if ((int64_t)m * batch == 0) return LOZA_OK;
  if (!rows || !cache || !pos0_dev) return fail(LOZA_ERR_INVALID, "NULL pointer");
  const int64_t esz = dtype == LOZA_BF16 ? 2 : 4;
  if ((d * esz) % 16 || !aligned16(rows) || !aligned16(cache) || (rows_stride_b * esz) % 16 ||
      (rows_stride_tok * esz) % 16 || (cache_stride_b * esz) % 16 || (cache_stride_tok * esz) % 16)
    return fail(LOZA_ERR_SHAPE, "ring append needs 16-byte rows, pointers and strides");
  return cuda_status(launch_ring_append(rows, rows_stride_b * esz, rows_stride_tok * esz, m, pos0_dev,
                                        pat.sink_blocks, pat.local_blocks, pat.block_size, cache, cache_stride_b * esz,
                                        cache_stride_tok * esz, batch, (int32_t)(d * esz), (cudaStream_t)stream),
                     "ring append launch");
}

loza_status_t ssa_decode_ring(const loza_attn_args_t* args, const int32_t* seq_lens_dev, loza_pattern_t pattern,
                              loza_stream_t stream) {
  g_last_error[0] = 0;
  if (args && args->batch == 0) return LOZA_OK;  // nothing to decode (seq_lens may be NULL)
  if (!seq_lens_dev) return fail(LOZA_ERR_INVALID, "seq_lens_dev is NULL");
  AttnProblem p;
  loza_status_t rc = make_problem(args, true, pattern, seq_lens_dev, &p);
  if (rc != LOZA_OK) return rc;
  if (args->n_kv != (int64_t)(pattern.sink_blocks + pattern.local_blocks) * pattern.block_size)
    return fail(LOZA_ERR_SHAPE, "ring cache: n_kv must be (s+l)*b");
  if ((int64_t)p.batch * p.heads == 0) return LOZA_OK;
  Path path;
  rc = choose_path(args, p, &path);
  if (rc != LOZA_OK) return rc;
  p.ring = 1;
  cudaError_t e;
  if (path != Path::kTc || !decode_pair_dispatch(p, nullptr, (cudaStream_t)stream, &e))
    return fail(LOZA_ERR_UNSUPPORTED, "ring decode: bf16, H <= 64, b %% 128 == 0, 2*batch <= SMs, v aliasing k");
  return cuda_status(e, "decode (ring) launch");
}

loza_status_t ssa_select_blocks(int64_t n_q, int64_t q_start, loza_pattern_t pat, int32_t causal, int32_t* idx_dev,
                                int32_t* count_dev, loza_stream_t stream) {
  g_last_error[0] = 0;
  if (pat.sink_blocks < 0 || pat.local_blocks < 1 || pat.block_size < 1) return fail(LOZA_ERR_INVALID, "bad pattern");
  if (causal != 1) return fail(LOZA_ERR_UNSUPPORTED, "SSA is causal only");
  if (n_q < 0 || q_start < 0 || q_start % pat.block_size) return fail(LOZA_ERR_SHAPE, "bad n_q / q_start");
  if (n_q == 0) return LOZA_OK;
  if (!idx_dev || !count_dev) return fail(LOZA_ERR_INVALID, "NULL output");
  return cuda_status(launch_select_blocks(n_q, q_start, pat.sink_blocks, pat.local_blocks, pat.block_size, idx_dev,
                                          count_dev, (cudaStream_t)stream),
                     "select_blocks launch");
}

size_t loza_seqpar_ws_bytes(const loza_attn_args_t* a, loza_pattern_t pat);

size_t loza_workspace_size(int32_t which, const loza_attn_args_t* a, loza_pattern_t pat, int32_t world) {
  (void)world;
  if (which == LOZA_WS_BLEND) return blend_ws_bytes();
  if (!a) return 0;
  AttnProblem p;
  if (which == LOZA_WS_BACKWARD) {
    if (make_problem(a, pat.local_blocks >= 1 && pat.block_size >= 1 && a->causal, pat, nullptr, &p) != LOZA_OK)
      return 0;
    return backward_ws_bytes(p);
  }
  if (which == LOZA_WS_DECODE || which == LOZA_WS_FULL_DECODE) {
    static const int32_t dummy = 1;
    if (make_problem(a, which == LOZA_WS_DECODE, pat, &dummy, &p) != LOZA_OK) return 0;
    if (a->in_dtype != LOZA_BF16) return 0;
    return decode_tc_ws_bytes(p);
  }
  if (which == LOZA_WS_SEQPAR) return loza_seqpar_ws_bytes(a, pat);
  return 0;
}

loza_status_t loza_workspace_init(int32_t which, const loza_attn_args_t* a, loza_pattern_t pat, int32_t world,
                                  void* ws, size_t ws_bytes, loza_stream_t stream) {
  g_last_error[0] = 0;
  const size_t need = loza_workspace_size(which, a, pat, world);
  if (need == 0) return LOZA_OK;
  if (!ws || ws_bytes < need) return fail(LOZA_ERR_INVALID, "workspace too small (%zu < %zu)", ws_bytes, need);
  return cuda_status(cudaMemsetAsync(ws, 0, need, (cudaStream_t)stream), "workspace init");
}

const char* loza_status_string(loza_status_t s) {
  switch (s) {
    case LOZA_OK: return "LOZA_OK";
    case LOZA_ERR_INVALID: return "LOZA_ERR_INVALID";
    case LOZA_ERR_SHAPE: return "LOZA_ERR_SHAPE";
    case LOZA_ERR_UNSUPPORTED: return "LOZA_ERR_UNSUPPORTED";
    case LOZA_ERR_CUDA: return "LOZA_ERR_CUDA";
    case LOZA_ERR_NCCL: return "LOZA_ERR_NCCL";
  }
  return "LOZA_ERR_UNKNOWN";
}

const char* loza_last_error(void) { return g_last_error; }
uint64_t loza_kernel_launches(void) { return g_launches.load(); }

int32_t loza_debug_force_kernel(const char* family, int32_t variant) {
  if (!family) return -1;
  if (strcmp(family, "decode") == 0 && variant >= 0 && variant <= 2) {
    g_knobs[kKnobDecode].store(variant);
    return 0;
  }
  if (strcmp(family, "backward") == 0 && variant >= 0 && variant <= 5) {
    g_knobs[kKnobBackward].store(variant);
    return 0;
  }
  return -1;
}
int32_t loza_num_sms(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

}  // extern "C"
