// Attention backward for SSA (Eq. 4) and full attention (Eq. 1): the chain rule of
// O_r = sum_j P_rj v_j, P_rj = exp(z_rj - LSE_r), z_rj = scale q_r . k_j over the allowed keys:
//   D_r = dO_r . O_r ;  dS_rj = P_rj (dO_r . v_j - D_r)
//   dQ_r = scale sum_j dS_rj k_j ;  dK_j = scale sum_r dS_rj q_r ;  dV_j = sum_r P_rj dO_r
// First GPU path: FFMA (SIMT), fp32 accumulation, recomputing P from the forward's LSE (no S matrix stored).
// Kernel 1 (a warp per query row): D_r and dQ_r over the row's allowed keys. Kernel 2 (a warp per key):
// dK_j and dV_j over the rows that attend key j (no atomics: deterministic). Dims are spread over the
// lanes (lane + 32 c), dot products are warp-reduced. The allowed sets are the closed form of the block
// selection (select_blocks.cu): sink blocks [0, s) and local blocks [max(s, QB - l + 1), QB], causal j <= p.
// Tiled variants below share staged rows across a CTA's warps (used when H % 8 == 0 and b % 16 == 0).
// The absorbed MLA shape in bf16 runs on the tensor cores instead (attn_bwd_mma.cu).
#include <math.h>
#include <stdlib.h>
#include <string.h>

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

// ---------------------------------------------------------------- tiled variants (H % 8 == 0, b % 16 == 0)
// The kernels above re-read every key row per query row and every query row per key. Here a CTA shares
// staged rows between its 8 warps, rows are staged with 16-byte vector loads (converted to fp32 in shared
// memory), and each lane owns dimension PAIRS d = 2 lane + 64 c (8-byte shared reads, two FMAs per read):
//  * rows: a CTA = the 8 heads h0 .. h0 + 7 of one token (identical key sets); keys are staged kKB at a time
//    and consumed by all 8 warps (one query row each).
//  * keys: a CTA = kKT = 16 keys of one b-block (identical attending row sets up to the per-key causal
//    bound); query rows (q, dO, LSE, D) are staged kRB at a time; each warp owns 2 keys (K/V and the dK/dV
//    accumulators in registers). Deterministic (no atomics).
constexpr int kKB = 8, kKT = 16, kRB = 8;
constexpr int kPQ = 9, kPV = 8;  // dimension pairs per lane: d_qk <= 576, d_v <= 512

// stage element range [0, d) of a row at `src + off` (elements) into dst[0, d) fp32; `tid`/`nth` split the
// work; vector path when the row start is 16-byte aligned and d spans whole 16-byte vectors
__device__ __forceinline__ void stage_row(float* dst, const void* src, int64_t off, int d, int bf16, int tid,
                                          int nth) {
  const int esz = bf16 ? 2 : 4, per = 16 / esz;
  const uint8_t* a = reinterpret_cast<const uint8_t*>(src) + off * esz;
  if (((reinterpret_cast<uintptr_t>(a) & 15) == 0) && d % per == 0) {
    for (int v = tid; v < d / per; v += nth) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(a) + v);
      if (bf16) {
        float4 lo, hi;
        lo.x = __uint_as_float(x.x << 16); lo.y = __uint_as_float(x.x & 0xFFFF0000u);
        lo.z = __uint_as_float(x.y << 16); lo.w = __uint_as_float(x.y & 0xFFFF0000u);
        hi.x = __uint_as_float(x.z << 16); hi.y = __uint_as_float(x.z & 0xFFFF0000u);
        hi.z = __uint_as_float(x.w << 16); hi.w = __uint_as_float(x.w & 0xFFFF0000u);
        reinterpret_cast<float4*>(dst)[2 * v] = lo;
        reinterpret_cast<float4*>(dst)[2 * v + 1] = hi;
      } else {
        reinterpret_cast<uint4*>(dst)[v] = x;
      }
    }
  } else {
    for (int e = tid; e < d; e += nth) dst[e] = ldf(src, off + e, bf16);
  }
}
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }

__global__ void __launch_bounds__(256) bwd_rows_tiled_kernel(BwdParams p, int v_alias) {
  extern __shared__ float sm[];  // [kKB][kstride]: d_qk (+ d_v unless V aliases K's first d_v columns)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rows = (int64_t)p.n_q * p.heads;
  const int64_t w0 = (int64_t)blockIdx.x * 8;
  const int64_t bi = w0 / rows, r0 = w0 - bi * rows;
  const int64_t t = r0 / p.heads, h = r0 - t * p.heads + warp;
  const int64_t pos = p.q_start + t;
  const int kstride = p.d_qk + (v_alias ? 0 : p.d_v);
  float2 qv[kPQ], dq[kPQ], dov[kPV];
  const int64_t qo = bi * p.q_sb + t * p.q_st + h * p.q_sh;
  const int64_t oo = bi * p.o_sb + t * p.o_st + h * p.o_sh;
  float Dp = 0.f;
#pragma unroll
  for (int c = 0; c < kPQ; ++c) {
    const int d = 2 * lane + 64 * c;
    qv[c] = d < p.d_qk ? make_float2(ldf(p.q, qo + d, p.in_bf16), ldf(p.q, qo + d + 1, p.in_bf16)) : make_float2(0.f, 0.f);
    dq[c] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int c = 0; c < kPV; ++c) {
    const int d = 2 * lane + 64 * c;
    if (d < p.d_v) {
      dov[c] = make_float2(ldf(p.dout, oo + d, p.out_bf16), ldf(p.dout, oo + d + 1, p.out_bf16));
      Dp = fmaf(dov[c].x, ldf(p.o, oo + d, p.out_bf16), fmaf(dov[c].y, ldf(p.o, oo + d + 1, p.out_bf16), Dp));
    } else {
      dov[c] = make_float2(0.f, 0.f);
    }
  }
  const float D = warp_sum(Dp);
  const float lse = p.lse[(bi * p.heads + h) * p.n_q + t];
  int64_t ja[2], jb[2];
  key_ranges(p, pos, ja[0], jb[0], ja[1], jb[1]);
  const int64_t na = jb[0] - ja[0], nk = na + (jb[1] - ja[1]);
  for (int64_t c0 = 0; c0 < nk; c0 += kKB) {
    const int nc = (int)(nk - c0 < kKB ? nk - c0 : kKB);
    // 32 threads per staged key row (warp kk stages key kk)
    if (warp < nc) {
      const int64_t f = c0 + warp, j = f < na ? ja[0] + f : ja[1] + (f - na);
      stage_row(sm + warp * kstride, p.k, bi * p.k_sb + j * p.k_st, p.d_qk, p.in_bf16, lane, 32);
      if (!v_alias) stage_row(sm + warp * kstride + p.d_qk, p.v, bi * p.v_sb + j * p.v_st, p.d_v, p.in_bf16, lane, 32);
    }
    __syncthreads();
    for (int kk = 0; kk < nc; ++kk) {
      const float* kr = sm + kk * kstride;
      const float* vr = v_alias ? kr : kr + p.d_qk;
      float2 k2[kPQ];
      float zp = 0.f, dpp = 0.f;
#pragma unroll
      for (int c = 0; c < kPQ; ++c) {
        const int d = 2 * lane + 64 * c;
        k2[c] = d < p.d_qk ? ld2(kr + d) : make_float2(0.f, 0.f);
        zp = fmaf(qv[c].x, k2[c].x, fmaf(qv[c].y, k2[c].y, zp));
      }
#pragma unroll
      for (int c = 0; c < kPV; ++c) {
        const int d = 2 * lane + 64 * c;
        if (d < p.d_v) {
          const float2 v2 = ld2(vr + d);
          dpp = fmaf(dov[c].x, v2.x, fmaf(dov[c].y, v2.y, dpp));
        }
      }
      const float z = warp_sum(zp) * p.scale, dP = warp_sum(dpp);
      const float P = expf(z - lse);
      const float dS = P * (dP - D) * p.scale;
#pragma unroll
      for (int c = 0; c < kPQ; ++c) {
        dq[c].x = fmaf(dS, k2[c].x, dq[c].x);
        dq[c].y = fmaf(dS, k2[c].y, dq[c].y);
      }
    }
    __syncthreads();
  }
  float* dqo = p.dq + ((bi * p.n_q + t) * p.heads + h) * p.d_qk;
#pragma unroll
  for (int c = 0; c < kPQ; ++c) {
    const int d = 2 * lane + 64 * c;
    if (d < p.d_qk) *reinterpret_cast<float2*>(dqo + d) = dq[c];
  }
  if (lane == 0) p.D[bi * rows + r0 + warp] = D;
}

__global__ void __launch_bounds__(256) bwd_keys_tiled_kernel(BwdParams p) {
  extern __shared__ float sm[];  // [kRB][d_qk + d_v] rows (q, dO), then lse[kRB], D[kRB]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = (p.n_kv + kKT - 1) / kKT;
  const int64_t bi = blockIdx.x / tiles, j0 = (blockIdx.x - bi * tiles) * kKT;
  const int rstride = p.d_qk + p.d_v;
  float* lse_s = sm + kRB * rstride;
  float* D_s = lse_s + kRB;
  int64_t jk[2];
  bool kvalid[2];
  float2 kv[2][kPQ], vv[2][kPV], dk[2][kPQ], dv[2][kPV];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    jk[e] = j0 + 2 * warp + e;
    kvalid[e] = jk[e] < p.n_kv;
    const int64_t jj = kvalid[e] ? jk[e] : 0;
    const int64_t ko = bi * p.k_sb + jj * p.k_st, vo = bi * p.v_sb + jj * p.v_st;
#pragma unroll
    for (int c = 0; c < kPQ; ++c) {
      const int d = 2 * lane + 64 * c;
      kv[e][c] = d < p.d_qk ? make_float2(ldf(p.k, ko + d, p.in_bf16), ldf(p.k, ko + d + 1, p.in_bf16))
                            : make_float2(0.f, 0.f);
      dk[e][c] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int c = 0; c < kPV; ++c) {
      const int d = 2 * lane + 64 * c;
      vv[e][c] = d < p.d_v ? make_float2(ldf(p.v, vo + d, p.in_bf16), ldf(p.v, vo + d + 1, p.in_bf16))
                           : make_float2(0.f, 0.f);
      dv[e][c] = make_float2(0.f, 0.f);
    }
  }
  // rows attending the tile's keys: causal pos >= j (per key below); SSA local block kb: blocks kb .. kb + l - 1
  int64_t p0 = p.causal ? j0 : 0, p1 = p.q_start + p.n_q;
  if (p.sparse) {
    const int64_t kb = j0 / p.b;
    if (kb >= p.s) {
      const int64_t pe = (kb + p.l) * (int64_t)p.b;
      if (pe < p1) p1 = pe;
    }
  }
  if (p0 < p.q_start) p0 = p.q_start;
  const int32_t nrow = p1 > p0 ? (int32_t)((p1 - p0) * p.heads) : 0;
  const int64_t rows = (int64_t)p.n_q * p.heads;
  const int32_t tq0 = (int32_t)(p0 - p.q_start), H = p.heads;
  for (int32_t rc = 0; rc < nrow; rc += kRB) {
    const int nr = nrow - rc < kRB ? nrow - rc : kRB;
    if (warp < nr) {  // warp rr stages row rr (q then dO)
      const int32_t ri = rc + warp, t = tq0 + ri / H, h = ri - (ri / H) * H;
      stage_row(sm + warp * rstride, p.q, bi * p.q_sb + (int64_t)t * p.q_st + (int64_t)h * p.q_sh, p.d_qk, p.in_bf16,
                lane, 32);
      stage_row(sm + warp * rstride + p.d_qk, p.dout, bi * p.o_sb + (int64_t)t * p.o_st + (int64_t)h * p.o_sh, p.d_v,
                p.out_bf16, lane, 32);
      if (lane == 0) {
        lse_s[warp] = p.lse[(bi * p.heads + h) * p.n_q + t];
        D_s[warp] = p.D[bi * rows + (int64_t)t * p.heads + h];
      }
    }
    __syncthreads();
    for (int rr = 0; rr < nr; ++rr) {
      const int64_t pos = p0 + (rc + rr) / H;
      const float* qr = sm + rr * rstride;
      const float* dor = qr + p.d_qk;
      float2 q2[kPQ], o2[kPV];
#pragma unroll
      for (int c = 0; c < kPQ; ++c) {
        const int d = 2 * lane + 64 * c;
        q2[c] = d < p.d_qk ? ld2(qr + d) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int c = 0; c < kPV; ++c) {
        const int d = 2 * lane + 64 * c;
        o2[c] = d < p.d_v ? ld2(dor + d) : make_float2(0.f, 0.f);
      }
      const float lse = lse_s[rr], Dr = D_s[rr];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (!kvalid[e] || (p.causal && pos < jk[e])) continue;  // warp-uniform
        float zp = 0.f, dpp = 0.f;
#pragma unroll
        for (int c = 0; c < kPQ; ++c) zp = fmaf(q2[c].x, kv[e][c].x, fmaf(q2[c].y, kv[e][c].y, zp));
#pragma unroll
        for (int c = 0; c < kPV; ++c) dpp = fmaf(o2[c].x, vv[e][c].x, fmaf(o2[c].y, vv[e][c].y, dpp));
        const float z = warp_sum(zp) * p.scale, dP = warp_sum(dpp);
        const float P = expf(z - lse);
        const float dS = P * (dP - Dr) * p.scale;
#pragma unroll
        for (int c = 0; c < kPQ; ++c) {
          dk[e][c].x = fmaf(dS, q2[c].x, dk[e][c].x);
          dk[e][c].y = fmaf(dS, q2[c].y, dk[e][c].y);
        }
#pragma unroll
        for (int c = 0; c < kPV; ++c) {
          dv[e][c].x = fmaf(P, o2[c].x, dv[e][c].x);
          dv[e][c].y = fmaf(P, o2[c].y, dv[e][c].y);
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    if (!kvalid[e]) continue;
    float* dko = p.dk + (bi * p.n_kv + jk[e]) * p.d_qk;
    float* dvo = p.dv + (bi * p.n_kv + jk[e]) * p.d_v;
#pragma unroll
    for (int c = 0; c < kPQ; ++c) {
      const int d = 2 * lane + 64 * c;
      if (d < p.d_qk) *reinterpret_cast<float2*>(dko + d) = dk[e][c];
    }
#pragma unroll
    for (int c = 0; c < kPV; ++c) {
      const int d = 2 * lane + 64 * c;
      if (d < p.d_v) *reinterpret_cast<float2*>(dvo + d) = dv[e][c];
    }
  }
}

// Key kernel with the query-row staging double-buffered by cp.async (16-byte global -> shared copies that
// need no registers): rows stay in their input format (bf16 or fp32) in shared memory and are converted at
// use, so chunk c + 1 streams from HBM while chunk c is computed (Q and dO of a long sequence do not fit
// in L2: the synchronous staging above exposed the DRAM latency every chunk). Used when every staged row
// is 16-byte aligned and whole 16-byte vectors long.
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <bool BF16>
__device__ __forceinline__ float2 raw2(const uint8_t* row, int d) {  // elements d, d + 1 of a staged row
  if (BF16) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(row + 2 * d);
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  }
  return *reinterpret_cast<const float2*>(row + 4 * d);
}

template <bool BF16>
__global__ void __launch_bounds__(256) bwd_keys_async_kernel(BwdParams p) {
  extern __shared__ __align__(16) uint8_t smb[];  // [2 buf][kRB][q bytes | dO bytes], then lse/D [2][kRB]
  constexpr int esz = BF16 ? 2 : 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = (p.n_kv + kKT - 1) / kKT;
  const int64_t bi = blockIdx.x / tiles, j0 = (blockIdx.x - bi * tiles) * kKT;
  const int qbytes = p.d_qk * esz, rbytes = qbytes + p.d_v * esz;
  float* lse_s = reinterpret_cast<float*>(smb + 2 * kRB * rbytes);
  float* D_s = lse_s + 2 * kRB;
  int64_t jk[2];
  bool kvalid[2];
  float2 kv[2][kPQ], vv[2][kPV], dk[2][kPQ], dv[2][kPV];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    jk[e] = j0 + 2 * warp + e;
    kvalid[e] = jk[e] < p.n_kv;
    const int64_t jj = kvalid[e] ? jk[e] : 0;
    const int64_t ko = bi * p.k_sb + jj * p.k_st, vo = bi * p.v_sb + jj * p.v_st;
#pragma unroll
    for (int c = 0; c < kPQ; ++c) {
      const int d = 2 * lane + 64 * c;
      kv[e][c] = d < p.d_qk ? make_float2(ldf(p.k, ko + d, p.in_bf16), ldf(p.k, ko + d + 1, p.in_bf16))
                            : make_float2(0.f, 0.f);
      dk[e][c] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int c = 0; c < kPV; ++c) {
      const int d = 2 * lane + 64 * c;
      vv[e][c] = d < p.d_v ? make_float2(ldf(p.v, vo + d, p.in_bf16), ldf(p.v, vo + d + 1, p.in_bf16))
                           : make_float2(0.f, 0.f);
      dv[e][c] = make_float2(0.f, 0.f);
    }
  }
  int64_t p0 = p.causal ? j0 : 0, p1 = p.q_start + p.n_q;
  if (p.sparse) {
    const int64_t kb = j0 / p.b;
    if (kb >= p.s) {
      const int64_t pe = (kb + p.l) * (int64_t)p.b;
      if (pe < p1) p1 = pe;
    }
  }
  if (p0 < p.q_start) p0 = p.q_start;
  const int32_t nrow = p1 > p0 ? (int32_t)((p1 - p0) * p.heads) : 0;
  const int64_t rows = (int64_t)p.n_q * p.heads;
  const int32_t tq0 = (int32_t)(p0 - p.q_start), H = p.heads;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smb);
  // issue chunk rc's copies into buffer bb (warp rr copies row rr: q then dO, 16 B per lane per step)
  auto issue = [&](int32_t rc, int bb) {
    const int nr = nrow - rc < kRB ? nrow - rc : kRB;
    if (warp < nr) {
      const int32_t ri = rc + warp, t = tq0 + ri / H, h = ri - (ri / H) * H;
      const uint8_t* qg = reinterpret_cast<const uint8_t*>(p.q) + (bi * p.q_sb + (int64_t)t * p.q_st + (int64_t)h * p.q_sh) * esz;
      const uint8_t* og = reinterpret_cast<const uint8_t*>(p.dout) + (bi * p.o_sb + (int64_t)t * p.o_st + (int64_t)h * p.o_sh) * esz;
      const uint32_t dst = sbase + (bb * kRB + warp) * rbytes;
      for (int v = lane; v < qbytes / 16; v += 32) cp_async16(dst + 16 * v, qg + 16 * v);
      for (int v = lane; v < (rbytes - qbytes) / 16; v += 32) cp_async16(dst + qbytes + 16 * v, og + 16 * v);
      if (lane == 0) {
        lse_s[bb * kRB + warp] = p.lse[(bi * p.heads + h) * p.n_q + t];
        D_s[bb * kRB + warp] = p.D[bi * rows + (int64_t)t * p.heads + h];
      }
    }
    cp_async_commit();
  };
  if (nrow > 0) issue(0, 0);
  int bb = 0;
  for (int32_t rc = 0; rc < nrow; rc += kRB, bb ^= 1) {
    const int nr = nrow - rc < kRB ? nrow - rc : kRB;
    if (rc + kRB < nrow) {
      issue(rc + kRB, bb ^ 1);  // the other buffer was released by the previous iteration's barrier
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncthreads();
    for (int rr = 0; rr < nr; ++rr) {
      const int64_t pos = p0 + (rc + rr) / H;
      const uint8_t* qr = smb + (bb * kRB + rr) * rbytes;
      const uint8_t* dor = qr + qbytes;
      float2 q2[kPQ], o2[kPV];
#pragma unroll
      for (int c = 0; c < kPQ; ++c) {
        const int d = 2 * lane + 64 * c;
        q2[c] = d < p.d_qk ? raw2<BF16>(qr, d) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int c = 0; c < kPV; ++c) {
        const int d = 2 * lane + 64 * c;
        o2[c] = d < p.d_v ? raw2<BF16>(dor, d) : make_float2(0.f, 0.f);
      }
      const float lse = lse_s[bb * kRB + rr], Dr = D_s[bb * kRB + rr];
      // both keys in one straight-line body (masked, not branched) so their dependency chains interleave;
      // each dot product in two partial sums
      float za[2] = {0.f, 0.f}, zb[2] = {0.f, 0.f}, pa[2] = {0.f, 0.f}, pb[2] = {0.f, 0.f};
#pragma unroll
      for (int c = 0; c < kPQ; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          za[e] = fmaf(q2[c].x, kv[e][c].x, za[e]);
          zb[e] = fmaf(q2[c].y, kv[e][c].y, zb[e]);
        }
#pragma unroll
      for (int c = 0; c < kPV; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          pa[e] = fmaf(o2[c].x, vv[e][c].x, pa[e]);
          pb[e] = fmaf(o2[c].y, vv[e][c].y, pb[e]);
        }
      float z[2] = {za[0] + zb[0], za[1] + zb[1]}, dP[2] = {pa[0] + pb[0], pa[1] + pb[1]};
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          z[e] += __shfl_xor_sync(0xffffffffu, z[e], o);
          dP[e] += __shfl_xor_sync(0xffffffffu, dP[e], o);
        }
      float P[2], dS[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool on = kvalid[e] && !(p.causal && pos < jk[e]);
        P[e] = on ? expf(z[e] * p.scale - lse) : 0.f;
        dS[e] = P[e] * (dP[e] - Dr) * p.scale;
      }
#pragma unroll
      for (int c = 0; c < kPQ; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          dk[e][c].x = fmaf(dS[e], q2[c].x, dk[e][c].x);
          dk[e][c].y = fmaf(dS[e], q2[c].y, dk[e][c].y);
        }
#pragma unroll
      for (int c = 0; c < kPV; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          dv[e][c].x = fmaf(P[e], o2[c].x, dv[e][c].x);
          dv[e][c].y = fmaf(P[e], o2[c].y, dv[e][c].y);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    if (!kvalid[e]) continue;
    float* dko = p.dk + (bi * p.n_kv + jk[e]) * p.d_qk;
    float* dvo = p.dv + (bi * p.n_kv + jk[e]) * p.d_v;
#pragma unroll
    for (int c = 0; c < kPQ; ++c) {
      const int d = 2 * lane + 64 * c;
      if (d < p.d_qk) *reinterpret_cast<float2*>(dko + d) = dk[e][c];
    }
#pragma unroll
    for (int c = 0; c < kPV; ++c) {
      const int d = 2 * lane + 64 * c;
      if (d < p.d_v) *reinterpret_cast<float2*>(dvo + d) = dv[e][c];
    }
  }
}

}  // namespace

static size_t d_bytes(const AttnProblem& a) {
  return (sizeof(float) * (size_t)a.batch * a.n_q * a.heads + 255) / 256 * 256;
}
// sink-tile partials, then the pair key kernels' local-tile row-split partials (short sequences)
static size_t part_bytes(const AttnProblem& a) {
  return (backward_mma_part_bytes(a) + 255) / 256 * 256 + (backward_local_part_bytes(a) + 255) / 256 * 256;
}
// D, then (tensor-core path, SSA) the sink-tile partials and the dS rows (attn_bwd_mma.cu / attn_bwd_tc.cu)
// (the dS rows only when the tcgen05 dS path can run: bf16 MLA shape, V aliasing K, packed rows)
size_t backward_ws_bytes(const AttnProblem& a) {
  const auto& kv = a.kv.seg[0];
  const bool v_alias = kv.v == kv.k && kv.v_st == kv.k_st && kv.v_sb == kv.k_sb;
  const bool ds_path = a.in_bf16 && a.out_bf16 && a.d_qk == 576 && a.d_v == 512 && v_alias &&
                       backward_tc_eligible(a, nullptr) && backward_ds_eligible(a);
  return d_bytes(a) + part_bytes(a) + (ds_path ? backward_ds_bytes(a) : 0);
}

cudaError_t launch_attn_backward(const AttnProblem& a, const void* dout, float* dq, float* dk, float* dv, void* ws,
                                 cudaStream_t st) {
  if (a.d_qk > 32 * kMaxCQ || a.d_v > 32 * kMaxCV) return cudaErrorNotSupported;
  // the absorbed MLA shape in bf16 runs on the tensor cores (test knob backward = 1 forces the FFMA kernels)
  if (knob(kKnobBackward) != 1 && backward_mma_eligible(a, dout))
    return launch_attn_backward_mma(
        a, dout, dq, dk, dv, reinterpret_cast<float*>(ws), reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + d_bytes(a)),
        backward_ws_bytes(a) > d_bytes(a) + part_bytes(a)
            ? reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(ws) + d_bytes(a) + part_bytes(a))
            : nullptr,
        st);
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
  // tiled paths: 8 heads per row CTA, 16-key tiles inside one b-block, dimension pairs (even d)
  const bool even = a.d_qk % 2 == 0 && a.d_v % 2 == 0;
  const bool tiled_rows = even && a.heads % 8 == 0, tiled_keys = even && (!a.sparse || a.b % kKT == 0);
  // V aliases K's first d_v columns (absorbed MLA: one latent row serves both)
  const int v_alias = p.v == p.k && p.v_st == p.k_st && p.v_sb == p.k_sb && a.d_v <= a.d_qk;
  if (rows > 0) {
    if (tiled_rows) {
      const size_t smem = sizeof(float) * kKB * (a.d_qk + (v_alias ? 0 : a.d_v));
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(bwd_rows_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      bwd_rows_tiled_kernel<<<(unsigned)(rows / 8), 256, smem, st>>>(p, v_alias);
    } else {
      bwd_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(p);
    }
    count_launch();
  }
  if (keys > 0) {
    const int64_t tiles = (a.n_kv + kKT - 1) / kKT;
    // cp.async staging: every q / dO row 16-byte aligned and whole vectors long (same dtype for q and dO)
    const int esz = a.in_bf16 ? 2 : 4;
    auto al = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
    const bool async_ok = tiled_keys && a.in_bf16 == a.out_bf16 && al(a.q) && al(dout) &&
                          (a.d_qk * esz) % 16 == 0 && (a.d_v * esz) % 16 == 0 && (a.q_sb * esz) % 16 == 0 &&
                          (a.q_st * esz) % 16 == 0 && (a.q_sh * esz) % 16 == 0 && (a.o_sb * esz) % 16 == 0 &&
                          (a.o_st * esz) % 16 == 0 && (a.o_sh * esz) % 16 == 0;
    if (async_ok) {
      const size_t smem = (size_t)2 * kRB * (a.d_qk + a.d_v) * esz + sizeof(float) * 4 * kRB;
      cudaError_t e = a.in_bf16 ? cudaFuncSetAttribute(bwd_keys_async_kernel<true>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                                : cudaFuncSetAttribute(bwd_keys_async_kernel<false>,
                                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      if (a.in_bf16)
        bwd_keys_async_kernel<true><<<(unsigned)(a.batch * tiles), 256, smem, st>>>(p);
      else
        bwd_keys_async_kernel<false><<<(unsigned)(a.batch * tiles), 256, smem, st>>>(p);
    } else if (tiled_keys) {
      const size_t smem = sizeof(float) * (kRB * (a.d_qk + a.d_v) + 2 * kRB);
      bwd_keys_tiled_kernel<<<(unsigned)(a.batch * tiles), 256, smem, st>>>(p);
    } else {
      bwd_keys_kernel<<<(unsigned)((keys + 7) / 8), 256, 0, st>>>(p);
    }
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace loza
