// Attention backward for SSA (Eq. 4) and full attention (Eq. 1): the chain rule of
// O_r = sum_j P_rj v_j, P_rj = exp(z_rj - LSE_r), z_rj = scale q_r . k_j over the allowed keys:
//   D_r = dO_r . O_r ;  dS_rj = P_rj (dO_r . v_j - D_r)
//   dQ_r = scale sum_j dS_rj k_j ;  dK_j = scale sum_r dS_rj q_r ;  dV_j = sum_r P_rj dO_r
// First GPU path: FFMA (SIMT), fp32 accumulation, recomputing P from the forward's LSE (no S matrix stored).
// Kernel 1 (a warp per query row): D_r and dQ_r over the row's allowed keys. Kernel 2 (a warp per key):
// dK_j and dV_j over the rows that attend key j (no atomics: deterministic). Dims are spread over the
// lanes (lane + 32 c), dot products are warp-reduced. The allowed sets are the closed form of the block
// selection (select_blocks.cu): sink blocks [0, s) and local blocks [max(s, QB - l + 1), QB], causal j <= p.
// Tensor-core version: a later round.
#include <math.h>

#include "internal.h"

namespace loza {

namespace {

constexpr int kMaxCQ = 18;  // d_qk <= 576
constexpr int kMaxCV = 16;  // d_v  <= 512

struct BwdParams {
  const void* q;
  const void* k;
  const void* v;
  const void* o;
  const void* dout;
  const float* lse;
  float* dq;
  float* dk;
  float* dv;
  float* D;  // workspace [B][n_q*H]
  int64_t q_sb, q_st, q_sh, k_sb, k_st, v_sb, v_st, o_sb, o_st, o_sh;
  int32_t batch, n_q, heads, d_qk, d_v;
  int64_t n_kv, q_start;
  int32_t in_bf16, out_bf16;
  float scale;
  int32_t sparse, causal, s, l, b;
};

__device__ __forceinline__ float ldf(const void* base, int64_t i, int bf16) {
  if (bf16) return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(base)[i] << 16);
  return reinterpret_cast<const float*>(base)[i];
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// keys of the query at absolute position p: [j0a, j1a) then [j0b, j1b)
__device__ __forceinline__ void key_ranges(const BwdParams& p, int64_t pos, int64_t& j0a, int64_t& j1a,
                                           int64_t& j0b, int64_t& j1b) {
  const int64_t last = p.causal ? (pos + 1 < p.n_kv ? pos + 1 : p.n_kv) : p.n_kv;
  if (!p.sparse) {
    j0a = 0;
    j1a = last;
    j0b = j1b = 0;
    return;
  }
  const int64_t QB = pos / p.b;
  int64_t se = (int64_t)p.s * p.b;
  if (se > last) se = last;
  int64_t lb = QB - p.l + 1;
  if (lb < p.s) lb = p.s;
  j0a = 0;
  j1a = se;
  j0b = lb * p.b;
  j1b = last;
  if (j0b < j1a) j0b = j1a;
  if (j1b < j0b) j1b = j0b;
}

__global__ void __launch_bounds__(256) bwd_rows_kernel(BwdParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)p.n_q * p.heads;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)p.batch * rows) return;
  const int64_t bi = w / rows, r = w - bi * rows;
  const int64_t t = r / p.heads, h = r - t * p.heads;
  const int64_t pos = p.q_start + t;
  float qv[kMaxCQ], dq[kMaxCQ], dov[kMaxCV];
  const int64_t qo = bi * p.q_sb + t * p.q_st + h * p.q_sh;
  const int64_t oo = bi * p.o_sb + t * p.o_st + h * p.o_sh;
  float Dp = 0.f;
#pragma unroll
  for (int c = 0; c < kMaxCQ; ++c) {
    const int d = lane + 32 * c;
    qv[c] = d < p.d_qk ? ldf(p.q, qo + d, p.in_bf16) : 0.f;
    dq[c] = 0.f;
  }
#pragma unroll
  for (int c = 0; c < kMaxCV; ++c) {
    const int d = lane + 32 * c;
    dov[c] = d < p.d_v ? ldf(p.dout, oo + d, p.out_bf16) : 0.f;
    if (d < p.d_v) Dp = fmaf(dov[c], ldf(p.o, oo + d, p.out_bf16), Dp);
  }
  const float D = warp_sum(Dp);
  const float lse = p.lse[(bi * p.heads + h) * p.n_q + t];
  int64_t ja[2], jb[2];
  key_ranges(p, pos, ja[0], jb[0], ja[1], jb[1]);
  for (int seg = 0; seg < 2; ++seg)
    for (int64_t j = ja[seg]; j < jb[seg]; ++j) {
      const int64_t ko = bi * p.k_sb + j * p.k_st, vo = bi * p.v_sb + j * p.v_st;
      float zp = 0.f, dpp = 0.f;
      float kv[kMaxCQ];
#pragma unroll
      for (int c = 0; c < kMaxCQ; ++c) {
        const int d = lane + 32 * c;
        kv[c] = d < p.d_qk ? ldf(p.k, ko + d, p.in_bf16) : 0.f;
        zp = fmaf(qv[c], kv[c], zp);
      }
#pragma unroll
      for (int c = 0; c < kMaxCV; ++c) {
        const int d = lane + 32 * c;
        if (d < p.d_v) dpp = fmaf(dov[c], ldf(p.v, vo + d, p.in_bf16), dpp);
      }
      const float z = warp_sum(zp) * p.scale, dP = warp_sum(dpp);
      const float P = expf(z - lse);
      const float dS = P * (dP - D) * p.scale;
#pragma unroll
      for (int c = 0; c < kMaxCQ; ++c) dq[c] = fmaf(dS, kv[c], dq[c]);
    }
  float* dqo = p.dq + ((bi * p.n_q + t) * p.heads + h) * p.d_qk;
#pragma unroll
  for (int c = 0; c < kMaxCQ; ++c) {
    const int d = lane + 32 * c;
    if (d < p.d_qk) dqo[d] = dq[c];
  }
  if (lane == 0) p.D[bi * rows + r] = D;
}

__global__ void __launch_bounds__(256) bwd_keys_kernel(BwdParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= (int64_t)p.batch * p.n_kv) return;
  const int64_t bi = w / p.n_kv, j = w - bi * p.n_kv;
  float kv[kMaxCQ], vv[kMaxCV], dk[kMaxCQ], dv[kMaxCV];
  const int64_t ko = bi * p.k_sb + j * p.k_st, vo = bi * p.v_sb + j * p.v_st;
#pragma unroll
  for (int c = 0; c < kMaxCQ; ++c) {
    const int d = lane + 32 * c;
    kv[c] = d < p.d_qk ? ldf(p.k, ko + d, p.in_bf16) : 0.f;
    dk[c] = 0.f;
  }
#pragma unroll
  for (int c = 0; c < kMaxCV; ++c) {
    const int d = lane + 32 * c;
    vv[c] = d < p.d_v ? ldf(p.v, vo + d, p.in_bf16) : 0.f;
    dv[c] = 0.f;
  }
  // query positions that attend key j: causal p >= j; SSA: sink key -> every later query, local key in block
  // kb -> queries in blocks kb .. kb + l - 1
  int64_t p0 = p.causal ? j : 0, p1 = p.q_start + p.n_q;
  if (p.sparse) {
    const int64_t kb = j / p.b;
    if (kb >= p.s) {
      const int64_t pe = (kb + p.l) * (int64_t)p.b;
      if (pe < p1) p1 = pe;
    }
  }
  if (p0 < p.q_start) p0 = p.q_start;
  const int64_t rows = (int64_t)p.n_q * p.heads;
  for (int64_t pos = p0; pos < p1; ++pos) {
    const int64_t t = pos - p.q_start;
    for (int64_t h = 0; h < p.heads; ++h) {
      const int64_t qo = bi * p.q_sb + t * p.q_st + h * p.q_sh;
      const int64_t oo = bi * p.o_sb + t * p.o_st + h * p.o_sh;
      float qv[kMaxCQ], dov[kMaxCV];
      float zp = 0.f, dpp = 0.f;
#pragma unroll
      for (int c = 0; c < kMaxCQ; ++c) {
        const int d = lane + 32 * c;
        qv[c] = d < p.d_qk ? ldf(p.q, qo + d, p.in_bf16) : 0.f;
        zp = fmaf(qv[c], kv[c], zp);
      }
#pragma unroll
      for (int c = 0; c < kMaxCV; ++c) {
        const int d = lane + 32 * c;
        dov[c] = d < p.d_v ? ldf(p.dout, oo + d, p.out_bf16) : 0.f;
        dpp = fmaf(dov[c], vv[c], dpp);
      }
      const float z = warp_sum(zp) * p.scale, dP = warp_sum(dpp);
      const float P = expf(z - p.lse[(bi * p.heads + h) * p.n_q + t]);
      const float dS = P * (dP - p.D[bi * rows + t * p.heads + h]) * p.scale;
#pragma unroll
      for (int c = 0; c < kMaxCQ; ++c) dk[c] = fmaf(dS, qv[c], dk[c]);
#pragma unroll
      for (int c = 0; c < kMaxCV; ++c) dv[c] = fmaf(P, dov[c], dv[c]);
    }
  }
  float* dko = p.dk + (bi * p.n_kv + j) * p.d_qk;
  float* dvo = p.dv + (bi * p.n_kv + j) * p.d_v;
#pragma unroll
  for (int c = 0; c < kMaxCQ; ++c) {
    const int d = lane + 32 * c;
    if (d < p.d_qk) dko[d] = dk[c];
  }
#pragma unroll
  for (int c = 0; c < kMaxCV; ++c) {
    const int d = lane + 32 * c;
    if (d < p.d_v) dvo[d] = dv[c];
  }
}

}  // namespace

size_t backward_ws_bytes(const AttnProblem& a) { return sizeof(float) * (size_t)a.batch * a.n_q * a.heads; }

cudaError_t launch_attn_backward(const AttnProblem& a, const void* dout, float* dq, float* dk, float* dv, void* ws,
                                 cudaStream_t st) {
  if (a.d_qk > 32 * kMaxCQ || a.d_v > 32 * kMaxCV) return cudaErrorNotSupported;
  BwdParams p;
  p.q = a.q;
  p.k = a.kv.seg[0].k;
  p.v = a.kv.seg[0].v;
  p.o = a.o;
  p.dout = dout;
  p.lse = a.lse;
  p.dq = dq;
  p.dk = dk;
  p.dv = dv;
  p.D = reinterpret_cast<float*>(ws);
  p.q_sb = a.q_sb;
  p.q_st = a.q_st;
  p.q_sh = a.q_sh;
  p.k_sb = a.kv.seg[0].k_sb;
  p.k_st = a.kv.seg[0].k_st;
  p.v_sb = a.kv.seg[0].v_sb;
  p.v_st = a.kv.seg[0].v_st;
  p.o_sb = a.o_sb;
  p.o_st = a.o_st;
  p.o_sh = a.o_sh;
  p.batch = a.batch;
  p.n_q = a.n_q;
  p.heads = a.heads;
  p.d_qk = a.d_qk;
  p.d_v = a.d_v;
  p.n_kv = a.n_kv;
  p.q_start = a.q_start;
  p.in_bf16 = a.in_bf16;
  p.out_bf16 = a.out_bf16;
  p.scale = a.scale;
  p.sparse = a.sparse;
  p.causal = a.causal;
  p.s = a.s;
  p.l = a.l;
  p.b = a.b;
  const int64_t rows = (int64_t)a.batch * a.n_q * a.heads, keys = (int64_t)a.batch * a.n_kv;
  if (rows > 0) {
    bwd_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(p);
    count_launch();
  }
  if (keys > 0) {
    bwd_keys_kernel<<<(unsigned)((keys + 7) / 8), 256, 0, st>>>(p);
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace loza
