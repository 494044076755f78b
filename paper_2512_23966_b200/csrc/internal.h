// Internal (non-ABI) declarations of libloza.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/loza.h"

namespace loza {

// A key/value sequence as up to 3 position-contiguous segments (plain prefill:
// one segment; sequence-parallel prefill: [sink | halo | shard]). Key at
// absolute position j lives in the segment with pos_begin <= j < pos_end, at
// row (j - pos_begin) of that segment.
struct KvSeg {
  int64_t pos_begin, pos_end;
  const void* k;
  const void* v;
  int64_t k_sb, k_st, v_sb, v_st;  // batch / token strides (elements)
};
struct KvView {
  int32_t nseg;
  KvSeg seg[3];
};

// fused calibration forward (ssa_prefill_blend): Eq. 3 applied in the SSA prefill epilogue
struct CalibArgs {
  const void* o_full;   // [B, n_q, H, d_v] bf16, o's layout
  const void* d_o_hat;  // same layout, nullable (forward only)
  const float* alpha;   // device scalar
  double* part;         // per-CTA fp64 partials of d_alpha (>= SM count entries), NULL without d_o_hat
  double* d_alpha;      // device scalar out, NULL without d_o_hat
  int32_t* status;      // nullable: LOZA_ERR_INVALID if alpha is not in [0, 1]
};

struct AttnProblem {
  int32_t batch, n_q, heads, d_qk, d_v;
  int64_t n_kv, q_start;
  int32_t in_bf16, out_bf16;
  float scale;
  int32_t causal, sparse;
  int32_t s, l, b;
  const void* q;
  int64_t q_sb, q_st, q_sh;
  void* o;
  int64_t o_sb, o_st, o_sh;
  float* lse;
  int64_t lse_sh;             // lse [B, H, *] head stride in elements (make_problem: n_q; a sub-range launch
                              // of a longer problem keeps the longer n_q)
  const int32_t* seq_lens;  // non-NULL => decode (one query at seq_len-1)
  KvView kv;
  const CalibArgs* calib = nullptr;  // non-NULL => fused blend epilogue (bf16 SSA prefill only)
  int32_t ring = 0;                  // decode: k/v is the bounded ring cache of ring_cache.cu (n_kv = (s+l)*b)
};

// launchers (return cudaError_t of the launch)
cudaError_t launch_select_blocks(int64_t n_q, int64_t q_start, int32_t s, int32_t l, int32_t b,
                                 int32_t* idx, int32_t* cnt, cudaStream_t st);
cudaError_t launch_attn_simt(const AttnProblem& p, cudaStream_t st);
cudaError_t launch_blend(const void* o_full, const void* o_sparse, const float* alpha, void* o_hat,
                         const void* d_o_hat, double* d_alpha, int64_t numel, int bf16, int32_t* status,
                         void* ws, cudaStream_t st);
size_t blend_ws_bytes();
// fixed-order fp64 sum of n per-CTA partials; NaN if alpha is not in [0, 1] (blend.cu)
cudaError_t launch_dalpha_reduce(const double* part, int n, const float* alpha, double* out, cudaStream_t st);
// tcgen05 paths (bf16, d_qk 576, d_v 512)
cudaError_t launch_prefill_tc(const AttnProblem& p, cudaStream_t st);
// non-absorbed (MHA) form, d_qk 192 / d_v 128, per-head K/V (k_sh, v_sh: head strides in elements)
// pair-cooperative SSA decode (attn_tc_decode_coop.cu): same eligibility as the pair kernel
cudaError_t launch_decode_coop(const AttnProblem& a, int32_t* status, cudaStream_t st);
// pair-cooperative eligibility: SSA, H == 64, b % 128 == 0, 2 * batch <= SMs
bool decode_coop_eligible(const AttnProblem& a, int sms);
// the SSA decode kernel for a problem the CTA-pair kernels take (coop for H == 64, key-split for H < 64; the
// decode test knob overrides); false if neither is eligible
bool decode_pair_dispatch(const AttnProblem& a, int32_t* status, cudaStream_t st, cudaError_t* err);
cudaError_t launch_prefill_mha(const AttnProblem& a, int64_t k_sh, int64_t v_sh, cudaStream_t st);
cudaError_t launch_decode_tc(const AttnProblem& p, void* ws, size_t ws_bytes, cudaStream_t st);
size_t decode_tc_ws_bytes(const AttnProblem& p);
// key-split pair SSA decode (attn_tc_decode_ks.cu): SSA, H <= 64, b % 128 == 0, V aliasing the KV rows,
// 2 * batch <= SMs; status (nullable) receives LOZA_ERR_SHAPE when a seq_len is clamped
constexpr size_t kDecodeStatusBytes = 256;
bool decode_ks_eligible(const AttnProblem& a, int sms);
cudaError_t launch_decode_ks(const AttnProblem& a, int32_t* status, cudaStream_t st);
size_t backward_ws_bytes(const AttnProblem& a);
// tensor-core backward (attn_bwd_mma.cu): bf16, d_qk 576, d_v 512, V = K[:, :512]; D [B][n_q*H] and the
// sink-tile partials (backward_mma_part_bytes) come from the backward workspace
bool backward_mma_eligible(const AttnProblem& a, const void* dout);
size_t backward_mma_part_bytes(const AttnProblem& a);
cudaError_t launch_attn_backward_mma(const AttnProblem& a, const void* dout, float* dq, float* dk, float* dv,
                                     float* D, float* part, uint16_t* ds, cudaStream_t st);
// tcgen05 key side of the backward (attn_bwd_tc.cu): dK, dV (or the sink-split partials) from D; needs the
// packed token x head row layout of q and d_o
bool backward_tc_eligible(const AttnProblem& a, const void* dout);
cudaError_t launch_bwd_dkdv_tc(const AttnProblem& a, const void* dout, float* dk, float* dv, const float* D,
                               float* part, uint16_t* ds, int nsplit, int n_sink, cudaStream_t st);
// SSA dS-row buffer [B][n_q*H][(s+l)*b] bf16 (written by the tcgen05 key kernel) and dQ = dS K on tcgen05
bool backward_ds_eligible(const AttnProblem& a);
bool backward_key64_eligible(const AttnProblem& a);
// d_ready (nullable): an event the dK kernel waits for (D computed on another stream, beside the dV kernel).
// With the dS row buffer and b == 128 the 128-key CTA-pair kernels run instead unless allow_pair is false.
// part_local: the pair kernels' local-tile row-split partials (backward_local_part_bytes), nullable when 0.
cudaError_t launch_bwd_key64_tc(const AttnProblem& a, const void* dout, float* dk, float* dv, const float* D,
                                float* part, uint16_t* ds, int nsplit, int n_sink, cudaStream_t st,
                                cudaEvent_t d_ready = nullptr, bool allow_pair = true, float* part_local = nullptr);
struct PairSplits {
  int nsplit, lsplit;  // row splits of each sink tile / each local tile
};
PairSplits backward_pair_splits(const AttnProblem& a);
int backward_local_splits(const AttnProblem& a);
size_t backward_local_part_bytes(const AttnProblem& a);
size_t backward_ds_bytes(const AttnProblem& a);
cudaError_t launch_bwd_D(const AttnProblem& a, const void* dout, float* D, cudaStream_t st);
// pair_keys: the key side ran the 128-key CTA-pair kernels (backward_pair_eligible), which write every slot of a
// row's visible blocks; dQ then runs on CTA pairs too when 256-row tiles stay inside one query block
cudaError_t launch_bwd_dq_tc(const AttnProblem& a, const uint16_t* ds, float* dq, cudaStream_t st, bool pair_keys);
// SSA with b == 128: the 128-key CTA-pair key kernels can take it (with the dS row buffer)
bool backward_pair_eligible(const AttnProblem& a);
cudaError_t launch_attn_backward(const AttnProblem& a, const void* dout, float* dq, float* dk, float* dv, void* ws,
                                 cudaStream_t st);
cudaError_t launch_ring_append(const void* rows, int64_t r_sb, int64_t r_st, int32_t m, const int32_t* pos0,
                               int32_t s, int32_t l, int32_t b, void* cache, int64_t c_sb, int64_t c_st,
                               int32_t batch, int32_t row_bytes, cudaStream_t st);

void count_launch(uint64_t n = 1);
// Test-only kernel overrides (loza_debug_force_kernel; never read from the environment): 0 = automatic choice.
// decode: 1 = pair-cooperative (H == 64 only), 2 = key-split pair. backward: 1 = FFMA kernels, 2 = warp-MMA key and
// row kernels, 3 = tcgen05 key kernel + warp-MMA row kernel for dQ.
enum KnobFamily { kKnobDecode = 0, kKnobBackward = 1, kNumKnobs = 2 };
int knob(KnobFamily f);
loza_status_t fail(loza_status_t st, const char* fmt, ...);
loza_status_t cuda_status(cudaError_t e, const char* what);
loza_status_t make_problem(const loza_attn_args_t* a, bool sparse, loza_pattern_t pat, const int32_t* seq_lens,
                           AttnProblem* p);
loza_status_t run_attention(const loza_attn_args_t* a, const AttnProblem& p, void* ws, size_t ws_bytes,
                            cudaStream_t st);
int device_sm_count();

}  // namespace loza

#include <cuda.h>
namespace loza {
// 3-D bf16 TMA map {d (contiguous), rows, batch}, box {64, box_rows, 1}, SWIZZLE_128B (tma_host.cu)
bool encode_3d(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t batch, int64_t row_stride_el,
               int64_t batch_stride_el, uint32_t box_rows);
bool encode_5d_heads(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t heads, uint64_t batch,
                     int64_t row_stride_el, int64_t head_stride_el, int64_t batch_stride_el, uint32_t box_rows,
                     uint32_t box_chunks);
bool encode_3d_f32(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t batch, int64_t row_stride_el,
                   int64_t batch_stride_el, uint32_t box_rows);
bool encode_4d_chunks(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t batch,
                      int64_t row_stride_el, int64_t batch_stride_el, uint32_t box_rows, uint32_t box_chunks);
}  // namespace loza
