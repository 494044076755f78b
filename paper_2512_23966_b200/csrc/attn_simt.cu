// SIMT fp32 attention (prefill / decode, SSA / full) for fp32 inputs.
//
// The fp32 configuration (BASELINE.json configs[0]: B1 H1 n1024 d64, (1,2,64))
// needs 1e-4 relative agreement with the fp64 oracle; tf32 tensor cores
// (10-bit mantissa) would miss it (DESIGN R14), so this path is plain FFMA.
// One warp per query row; keys are visited only inside the allowed ranges of
// Eq. 4 (sink range [0, s*b) and the local range [(QB-l+1)*b, p], both clipped
// to j <= p), 32 at a time: each lane computes one logit, the warp does an
// online-softmax update (running max / sum) and every lane accumulates its
// d_v/32 output columns.
#include "internal.h"

namespace loza {

namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int kMaxD = 576;
constexpr int kMaxVPerLane = 16;  // d_v <= 512

__device__ __forceinline__ float ld_in(const void* base, int64_t off, int bf16) {
  if (bf16) {
    const unsigned short u = reinterpret_cast<const unsigned short*>(base)[off];
    return __uint_as_float(((unsigned)u) << 16);
  }
  return reinterpret_cast<const float*>(base)[off];
}

__device__ __forceinline__ const KvSeg* find_seg(const KvView& kv, int64_t j) {
  const KvSeg* s = &kv.seg[0];
#pragma unroll
  for (int i = 1; i < 3; ++i)
    if (i < kv.nseg && j >= kv.seg[i].pos_begin) s = &kv.seg[i];
  return s;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct RowState {
  float m, l;
  float acc[kMaxVPerLane];
};

__device__ __forceinline__ void visit_range(const AttnProblem& p, const float* qs, int bi, int64_t j_begin,
                                            int64_t j_end, RowState& st, int lane) {
  for (int64_t j0 = j_begin; j0 < j_end; j0 += 32) {
    const int64_t j = j0 + lane;
    float logit = -INFINITY;
    if (j < j_end) {
      const KvSeg* sg = find_seg(p.kv, j);
      const int64_t koff = bi * sg->k_sb + (j - sg->pos_begin) * sg->k_st;
      float acc = 0.f;
      for (int d = 0; d < p.d_qk; ++d) acc = fmaf(qs[d], ld_in(sg->k, koff + d, p.in_bf16), acc);
      logit = acc * p.scale;
    }
    const float m_new = fmaxf(st.m, warp_max(logit));
    const float corr = expf(st.m - m_new);  // st.m = -inf on the first chunk -> 0
    const float pj = (j < j_end) ? expf(logit - m_new) : 0.f;
    st.l = st.l * corr + warp_sum(pj);
#pragma unroll
    for (int c = 0; c < kMaxVPerLane; ++c) st.acc[c] *= corr;
    const int nvalid = (int)(j_end - j0 < 32 ? j_end - j0 : 32);
    for (int t = 0; t < nvalid; ++t) {
      const float w = __shfl_sync(0xffffffffu, pj, t);
      const int64_t jj = j0 + t;
      const KvSeg* sg = find_seg(p.kv, jj);
      const int64_t voff = bi * sg->v_sb + (jj - sg->pos_begin) * sg->v_st;
#pragma unroll
      for (int c = 0; c < kMaxVPerLane; ++c) {
        const int d = lane + 32 * c;
        if (d < p.d_v) st.acc[c] = fmaf(w, ld_in(sg->v, voff + d, p.in_bf16), st.acc[c]);
      }
    }
    st.m = m_new;
  }
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) attn_simt_kernel(const AttnProblem p) {
  __shared__ float qsm[kWarpsPerBlock][kMaxD];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + wib;
  const int64_t rows = (int64_t)p.batch * p.n_q * p.heads;
  if (row >= rows) return;
  const int h = (int)(row % p.heads);
  const int64_t ti = row / p.heads;
  const int i = (int)(ti % p.n_q);
  const int bi = (int)(ti / p.n_q);

  int64_t pos, n_keys;
  if (p.seq_lens) {
    int64_t sl = p.seq_lens[bi];
    sl = sl < 1 ? 1 : (sl > p.n_kv ? p.n_kv : sl);
    pos = sl - 1;
    n_keys = sl;
  } else {
    pos = p.q_start + i;
    n_keys = p.n_kv;
  }
  float* qs = qsm[wib];
  const int64_t qoff = bi * p.q_sb + (int64_t)i * p.q_st + (int64_t)h * p.q_sh;
  for (int d = lane; d < p.d_qk; d += 32) qs[d] = ld_in(p.q, qoff + d, p.in_bf16);
  __syncwarp();

  RowState st;
  st.m = -INFINITY;
  st.l = 0.f;
#pragma unroll
  for (int c = 0; c < kMaxVPerLane; ++c) st.acc[c] = 0.f;

  const int64_t causal_end = p.causal ? pos + 1 : n_keys;
  if (!p.sparse) {
    visit_range(p, qs, bi, 0, causal_end, st, lane);
  } else {
    const int64_t qb = pos / p.b;
    const int64_t sink_end = ((int64_t)p.s * p.b < causal_end ? (int64_t)p.s * p.b : causal_end);
    int64_t loc_begin = (qb - p.l + 1) * (int64_t)p.b;
    if (loc_begin < (int64_t)p.s * p.b) loc_begin = (int64_t)p.s * p.b;
    visit_range(p, qs, bi, 0, sink_end, st, lane);
    visit_range(p, qs, bi, loc_begin, causal_end, st, lane);
  }

  const float inv = 1.f / st.l;
  const int64_t ooff = bi * p.o_sb + (int64_t)i * p.o_st + (int64_t)h * p.o_sh;
#pragma unroll
  for (int c = 0; c < kMaxVPerLane; ++c) {
    const int d = lane + 32 * c;
    if (d < p.d_v) {
      const float v = st.acc[c] * inv;
      if (p.out_bf16) {
        unsigned u = __float_as_uint(v);
        u = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
        reinterpret_cast<unsigned short*>(p.o)[ooff + d] = (unsigned short)u;
      } else {
        reinterpret_cast<float*>(p.o)[ooff + d] = v;
      }
    }
  }
  if (p.lse && lane == 0) p.lse[((int64_t)bi * p.heads + h) * p.lse_sh + i] = st.m + logf(st.l);
}

}  // namespace

cudaError_t launch_attn_simt(const AttnProblem& p, cudaStream_t st) {
  const int64_t rows = (int64_t)p.batch * p.n_q * p.heads;
  if (rows == 0) return cudaSuccess;
  const int64_t blocks = (rows + kWarpsPerBlock - 1) / kWarpsPerBlock;
  attn_simt_kernel<<<(unsigned)blocks, kWarpsPerBlock * 32, 0, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza
