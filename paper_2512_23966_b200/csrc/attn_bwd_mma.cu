// Attention backward on the tensor cores: the gradients of Eq. 4 (SSA) or Eq. 1 (full
// attention), as defined in attn_bwd_simt.cu's header,
//   D_r = dO_r . O_r ;  P_rj = exp(scale q_r . k_j - LSE_r) ;  dS_rj = P_rj (dO_r . v_j - D_r)
//   dQ_r = scale sum_j dS_rj k_j ;  dK_j = scale sum_r dS_rj q_r ;  dV_j = sum_r P_rj dO_r
// for the absorbed MLA shape (bf16, d_qk 576, d_v 512, V = the first 512 columns of the latent row K), with
// warp-level mma.sync m16n8k16 (bf16 operands, fp32 accumulators): the dK / dV accumulators of a key tile
// (32 keys x 1088 fp32 = 139 KB) spread over 8 warps' registers. The first tensor-core backward; the default
// is now attn_bwd_tc.cu (tcgen05, accumulators transposed in TMEM) where its layout conditions hold.
// Deterministic, no atomics:
//  - row kernel: 64 query rows (flattened token x head, one key set per token) per CTA; Q / dO rows resident
//    in shared memory, 32-key K tiles double-buffered with cp.async; S, dP -> dS (bf16, shared) -> dQ += dS K
//    (fp32 accumulators in registers, 144 per thread); D_r in the prologue (also written for the key kernel).
//  - key kernel: 32 keys of one b-block per CTA (K resident), the rows that attend them streamed as
//    32-row Q / dO tiles (cp.async, double-buffered); S^T, dP^T -> P^T, dS^T (bf16, shared) ->
//    [dK | dV] += [dS^T Q | P^T dO] (136 fp32 accumulators per thread). The sink key tiles of SSA are
//    attended by every row: their row range is split over `nsplit` CTAs whose fp32 partials are summed in a
//    fixed order by a third kernel.
// P and dS are rounded to bf16 as MMA operands (fp32 softmax arithmetic); bf16-path tolerance as the forward.
// Shared-memory rows are padded by 16 B (ldmatrix conflict-free).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "internal.h"

namespace loza {

namespace {

constexpr int kDQK = 576, kDV = 512, kDKV = kDQK + kDV;
constexpr int kQRow = kDQK * 2 + 16;  // 1168 B
constexpr int kORow = kDV * 2 + 16;   // 1040 B
constexpr int kTRow = 32 * 2 + 16;    // 80 B: a 32-wide bf16 tile row
constexpr float kLog2e = 1.4426950408889634f;

// row kernel shared memory
constexpr int kRRows = 64, kRKeys = 32;
constexpr int kROffQ = 0;
constexpr int kROffDO = kROffQ + kRRows * kQRow;
constexpr int kROffK = kROffDO + kRRows * kORow;
constexpr int kROffDS = kROffK + 2 * kRKeys * kQRow;
constexpr int kROffL = kROffDS + kRRows * kTRow;
constexpr int kROffD = kROffL + kRRows * 4;
constexpr int kRSmem = kROffD + kRRows * 4;
// key kernel shared memory
constexpr int kKKeys = 32, kKRows = 32;
constexpr int kKOffK = 0;
constexpr int kKOffQ = kKOffK + kKKeys * kQRow;
constexpr int kKOffDO = kKOffQ + 2 * kKRows * kQRow;
constexpr int kKOffP = kKOffDO + 2 * kKRows * kORow;
constexpr int kKOffDS = kKOffP + kKKeys * kTRow;
constexpr int kKOffL = kKOffDS + kKKeys * kTRow;
constexpr int kKOffD = kKOffL + 2 * kKRows * 4;
constexpr int kKOffPos = kKOffD + 2 * kKRows * 4;  // int [2][32]: the row's position
constexpr int kKOffLb = kKOffPos + 2 * kKRows * 4;  // int [2][32]: its first local block pos / b - l + 1
constexpr int kPartRow = 40;                         // fp32 per partial row (32 + pad: float2 stores conflict-free)
constexpr int kKOffPart = kKOffLb + 2 * kKRows * 4;  // fp32 [2 (S, dP)][4 k quarters][32 keys][kPartRow]
constexpr int kKSmem = kKOffPart + 2 * 4 * kKKeys * kPartRow * 4;
static_assert(kRSmem <= 227 * 1024 && kKSmem <= 227 * 1024, "shared memory");

struct MP {
  const uint16_t* q;
  const uint16_t* k;  // V = k[:, :512]
  const uint16_t* o;
  const uint16_t* dout;
  const float* lse;
  float* dq;
  float* dk;
  float* dv;
  float* D;     // [B][n_q * H]
  float* part;  // sink-tile partials [B][n_sink][nsplit][32][1088]
  int64_t q_sb, q_st, q_sh, k_sb, k_st, o_sb, o_st, o_sh;
  int32_t batch, n_q, heads, n_kv, q_start;
  float scale, sl2;
  int32_t sparse, causal, s, l, b;
  int32_t nsplit, n_sink;
  uint32_t h_m, h_p;  // n / heads = (n * h_m) >> h_p, exact for n < 2^31
};

__host__ void fastdiv_init(uint32_t d, uint32_t& m, uint32_t& sh) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  sh = 31 + l;
  m = (uint32_t)(((1ull << sh) + d - 1) / d);
}
__device__ __forceinline__ int div_h(const MP& p, int n) { return (int)(((uint64_t)(uint32_t)n * p.h_m) >> p.h_p); }

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm4t(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
// D (16x8 fp32) += A (16x16 bf16, row) * B (16x8 bf16, col)
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v)); }

// The selection rule of attn_bwd_simt.cu's key_ranges as a predicate, for the query at position pos and key j:
//   j < n_kv  and  (not causal or j <= pos)  and  (dense or j / b < s or j / b >= pos / b - l + 1),
// evaluated below with the key block hoisted per tile and the row terms precomputed.
__device__ __forceinline__ int last_key(const MP& p, int pos) {
  return p.causal ? (pos + 1 < p.n_kv ? pos + 1 : p.n_kv) : p.n_kv;
}

// ---------------------------------------------------------------------------------------------- row kernel
__global__ void __launch_bounds__(256, 1) bwd_dq_mma_kernel(MP p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int H = p.heads, rows = p.n_q * H;
  const int rtiles = (rows + kRRows - 1) / kRRows;
  const int bi = blockIdx.x / rtiles, r0 = (blockIdx.x - bi * rtiles) * kRRows;
  const int nr = rows - r0 < kRRows ? rows - r0 : kRRows;
  float* lse_s = reinterpret_cast<float*>(smem + kROffL);
  float* D_s = reinterpret_cast<float*>(smem + kROffD);
  // Q and dO rows (zero-filled past the last row)
  for (int i = tid; i < kRRows * (kDQK / 8); i += 256) {
    const int ri = i / (kDQK / 8), c = i - ri * (kDQK / 8);
    const bool v = ri < nr;
    const int r = v ? r0 + ri : 0, t = div_h(p, r), h = r - t * H;
    cp16(sb + kROffQ + ri * kQRow + 16 * c, p.q + bi * p.q_sb + (int64_t)t * p.q_st + (int64_t)h * p.q_sh + 8 * c, v);
  }
  for (int i = tid; i < kRRows * (kDV / 8); i += 256) {
    const int ri = i / (kDV / 8), c = i - ri * (kDV / 8);
    const bool v = ri < nr;
    const int r = v ? r0 + ri : 0, t = div_h(p, r), h = r - t * H;
    cp16(sb + kROffDO + ri * kORow + 16 * c, p.dout + bi * p.o_sb + (int64_t)t * p.o_st + (int64_t)h * p.o_sh + 8 * c, v);
  }
  cp_commit();
  // key ranges: the union over the tile's tokens (first P0, last P1) of [0, se) and [j0b, j1b); each range's
  // own bounds are part of the mask so the two never count a key twice
  const int P0 = p.q_start + r0 / H, P1 = p.q_start + (r0 + nr - 1) / H;
  int lo[2], hi[2];
  {
    const int last = last_key(p, P1);
    if (!p.sparse) {
      lo[0] = 0;
      hi[0] = last;
      lo[1] = hi[1] = 0;
    } else {
      int se = p.s * p.b;
      if (se > last) se = last;
      int lb = P0 / p.b - p.l + 1;
      if (lb < p.s) lb = p.s;
      lo[0] = 0;
      hi[0] = se;
      lo[1] = lb * p.b;
      if (lo[1] < se) lo[1] = se;
      hi[1] = last > lo[1] ? last : lo[1];
    }
  }
  const int nt0 = (hi[0] - lo[0] + kRKeys - 1) / kRKeys, ntiles = nt0 + (hi[1] - lo[1] + kRKeys - 1) / kRKeys;
  auto tile_j0 = [&](int it) { return it < nt0 ? lo[0] + it * kRKeys : lo[1] + (it - nt0) * kRKeys; };
  auto issue_k = [&](int it, int buf) {
    const int j0 = tile_j0(it);
    {  // 8 threads per key row, 9 chunks each
      const int kj = tid >> 3, c0 = tid & 7, j = j0 + kj;
      const bool v = j < p.n_kv;
      const uint16_t* kg = p.k + bi * p.k_sb + (int64_t)(v ? j : 0) * p.k_st + 8 * c0;
      const uint32_t ks = sb + kROffK + (buf * kRKeys + kj) * kQRow + 16 * c0;
#pragma unroll
      for (int u = 0; u < kDQK / 64; ++u) cp16(ks + 128 * u, kg + 64 * u, v);
    }
    cp_commit();
  };
  if (ntiles > 0) issue_k(0, 0);
  if (tid < kRRows) {
    const bool v = tid < nr;
    const int r = v ? r0 + tid : 0, t = r / H, h = r - t * H;
    lse_s[tid] = v ? p.lse[((int64_t)bi * H + h) * p.n_q + t] * kLog2e : 0.f;
  }
  cp_wait<0>();
  __syncthreads();
  // D_r = dO_r . O_r (fp32), 8 rows per warp
  for (int ri = warp * 8; ri < warp * 8 + 8; ++ri) {
    float acc = 0.f;
    if (ri < nr) {
      const int r = r0 + ri, t = r / H, h = r - t * H;
      const uint16_t* orow = p.o + bi * p.o_sb + (int64_t)t * p.o_st + (int64_t)h * p.o_sh;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int c = lane + 32 * u;
        const uint4 ov = *reinterpret_cast<const uint4*>(orow + 8 * c);
        const uint4 dv = *reinterpret_cast<const uint4*>(smem + kROffDO + ri * kORow + 16 * c);
        const uint32_t oa[4] = {ov.x, ov.y, ov.z, ov.w}, da[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          acc = fmaf(__uint_as_float(oa[e] << 16), __uint_as_float(da[e] << 16), acc);
          acc = fmaf(__uint_as_float(oa[e] & 0xFFFF0000u), __uint_as_float(da[e] & 0xFFFF0000u), acc);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      D_s[ri] = acc;
      if (ri < nr) p.D[(int64_t)bi * rows + r0 + ri] = acc;
    }
  }
  __syncthreads();
  const int mrow = 16 * (warp & 3), ncol = 16 * (warp >> 2), dh = 288 * (warp >> 2);
  // this thread's two C-fragment rows
  int posr[2], lbr[2];
  float lser[2], Dr[2];
  bool rv[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int ri = mrow + g + 8 * u;
    rv[u] = ri < nr;
    posr[u] = p.q_start + div_h(p, r0 + (rv[u] ? ri : 0));
    lbr[u] = posr[u] / p.b - p.l + 1;
    lser[u] = lse_s[ri];
    Dr[u] = D_s[ri];
  }
  float acc[36][4];
#pragma unroll
  for (int n = 0; n < 36; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
  const uint32_t aQ = sb + kROffQ + (mrow + (lane & 15)) * kQRow + (lane >> 4) * 16;
  const uint32_t aO = sb + kROffDO + (mrow + (lane & 15)) * kORow + (lane >> 4) * 16;
  const uint32_t bK = ((lane & 7) + ((lane >> 4) << 3) + ncol) * kQRow + ((lane >> 3) & 1) * 16;
  const uint32_t aS = sb + kROffDS + (mrow + (lane & 15)) * kTRow + (lane >> 4) * 16;
  const uint32_t bKt = ((lane & 7) + ((lane >> 3) & 1) * 8) * kQRow + (lane >> 4) * 16 + 2 * dh;
  for (int it = 0; it < ntiles; ++it) {
    const int buf = it & 1;
    if (it + 1 < ntiles) issue_k(it + 1, buf ^ 1);
    const uint32_t kbase = sb + kROffK + buf * kRKeys * kQRow;
    // two independent chains per 8-key tile (even / odd k steps), summed afterwards
    float s4[4][4] = {}, d4[4][4] = {};
#pragma unroll 3
    for (int kk = 0; kk < kDQK / 16; kk += 2) {
      uint32_t a[4], b[4], a2[4], b2[4];
      ldsm4(aQ + 32 * kk, a);
      ldsm4(kbase + bK + 32 * kk, b);
      ldsm4(aQ + 32 * kk + 32, a2);
      ldsm4(kbase + bK + 32 * kk + 32, b2);
      mma(s4[0], a, b[0], b[1]);
      mma(s4[1], a, b[2], b[3]);
      mma(s4[2], a2, b2[0], b2[1]);
      mma(s4[3], a2, b2[2], b2[3]);
    }
#pragma unroll 4
    for (int kk = 0; kk < kDV / 16; kk += 2) {
      uint32_t a[4], b[4], a2[4], b2[4];
      ldsm4(aO + 32 * kk, a);
      ldsm4(kbase + bK + 32 * kk, b);
      ldsm4(aO + 32 * kk + 32, a2);
      ldsm4(kbase + bK + 32 * kk + 32, b2);
      mma(d4[0], a, b[0], b[1]);
      mma(d4[1], a, b[2], b[3]);
      mma(d4[2], a2, b2[0], b2[1]);
      mma(d4[3], a2, b2[2], b2[3]);
    }
    float s[2][4], dp[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s[nt][e] = s4[nt][e] + s4[nt + 2][e];
        dp[nt][e] = d4[nt][e] + d4[nt + 2][e];
      }
    const int j0 = tile_j0(it), rlo = it < nt0 ? lo[0] : lo[1], rhi = it < nt0 ? hi[0] : hi[1];
    // the tile lies in one b-block (b % 32 == 0; range starts are block-aligned): allowed() once per tile
    const int kbt = j0 / p.b;
    const bool tsink = !p.sparse || kbt < p.s;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        float ds2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = j0 + ncol + 8 * nt + 2 * t4 + e;
          const bool ok = rv[u] && j >= rlo && j < rhi && j < p.n_kv && (!p.causal || j <= posr[u]) &&
                          (tsink || kbt >= lbr[u]);
          const float pv = ok ? ex2f(fmaf(s[nt][2 * u + e], p.sl2, -lser[u])) : 0.f;
          ds2[e] = pv * (dp[nt][2 * u + e] - Dr[u]);
        }
        sts32(sb + kROffDS + (mrow + g + 8 * u) * kTRow + (ncol + 8 * nt + 2 * t4) * 2, pack2(ds2[0], ds2[1]));
      }
    }
    __syncthreads();  // dS tile complete
    uint32_t a0[4], a1[4];
    ldsm4(aS, a0);
    ldsm4(aS + 32, a1);
#pragma unroll
    for (int np = 0; np < 18; ++np) {
      uint32_t b[4];
      ldsm4t(kbase + bKt + 32 * np, b);
      mma(acc[2 * np], a0, b[0], b[1]);
      mma(acc[2 * np + 1], a0, b[2], b[3]);
      ldsm4t(kbase + bKt + 16 * kQRow + 32 * np, b);
      mma(acc[2 * np], a1, b[0], b[1]);
      mma(acc[2 * np + 1], a1, b[2], b[3]);
    }
    cp_wait<0>();
    __syncthreads();  // next K tile landed; this tile's K / dS reads done
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    if (!rv[u]) continue;
    float* out = p.dq + ((int64_t)bi * rows + r0 + mrow + g + 8 * u) * kDQK + dh + 2 * t4;
#pragma unroll
    for (int n = 0; n < 36; ++n)
      *reinterpret_cast<float2*>(out + 8 * n) = make_float2(acc[n][2 * u] * p.scale, acc[n][2 * u + 1] * p.scale);
  }
}

// ---------------------------------------------------------------------------------------------- key kernel
__global__ void __launch_bounds__(256, 1) bwd_dkdv_mma_kernel(MP p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int H = p.heads;
  const int ktiles = (p.n_kv + kKKeys - 1) / kKKeys;
  const int bi = blockIdx.x / ktiles, tile = blockIdx.x - bi * ktiles, j0 = tile * kKKeys;
  // rows attending keys [j0, j0 + 32) (one b-block): positions [p0, p1)
  int p0 = p.causal ? j0 : 0, p1 = p.q_start + p.n_q;
  const int kb = j0 / p.b;
  if (p.sparse && kb >= p.s) {
    const int pe = (kb + p.l) * p.b;
    if (pe < p1) p1 = pe;
  }
  if (p0 < p.q_start) p0 = p.q_start;
  int R0 = 0, R1 = 0;
  if (p1 > p0) {
    R0 = (p0 - p.q_start) * H;
    R1 = (p1 - p.q_start) * H;
  }
  const bool split = p.sparse && kb < p.s && p.nsplit > 1;
  if (split) {
    const int chunk = ((R1 - R0 + p.nsplit - 1) / p.nsplit + kKRows - 1) / kKRows * kKRows;
    const int a = R0 + (int)blockIdx.y * chunk, e = a + chunk;
    R0 = a < R1 ? a : R1;
    R1 = e < R1 ? e : R1;
  } else if (blockIdx.y > 0) {
    return;
  }
  float* lse_s = reinterpret_cast<float*>(smem + kKOffL);
  float* D_s = reinterpret_cast<float*>(smem + kKOffD);
  int* pos_s = reinterpret_cast<int*>(smem + kKOffPos);
  int* lb_s = reinterpret_cast<int*>(smem + kKOffLb);
  for (int i = tid; i < kKKeys * (kDQK / 8); i += 256) {
    const int kj = i / (kDQK / 8), c = i - kj * (kDQK / 8);
    const int j = j0 + kj;
    const bool v = j < p.n_kv;
    cp16(sb + kKOffK + kj * kQRow + 16 * c, p.k + bi * p.k_sb + (int64_t)(v ? j : 0) * p.k_st + 8 * c, v);
  }
  cp_commit();
  // Row tiles in segments. A local (SSA) key tile's rows span <= l query blocks; they are taken block by
  // block in the order m mod l, so at step sigma every such CTA reads query block m = sigma (mod l): the ~4 l
  // CTAs whose windows hold a block read it at about the same time (L2 reuse of the Q / dO stream).
  const int L = p.sparse && !split && kb >= p.s ? p.l : 1;
  const int m0 = p0 / p.b, m1 = (p1 - 1) / p.b;
  auto next_seg = [&](int& sig, int& rb, int& re) {  // the first non-empty segment after sig (sig = L: none)
    while (++sig < L) {
      if (L == 1) {
        rb = R0;
        re = R1;
      } else {
        const int m = m0 + ((sig - m0) % L + L) % L;
        if (m > m1) continue;
        const int a = m * p.b > p0 ? m * p.b : p0, e = (m + 1) * p.b < p1 ? (m + 1) * p.b : p1;
        rb = (a - p.q_start) * H;
        re = (e - p.q_start) * H;
      }
      if (rb < re) return;
    }
  };
  auto advance = [&](int& sig, int& rb, int& re) {
    rb += kKRows;
    if (rb >= re) next_seg(sig, rb, re);
  };
  const int rows = p.n_q * H;
  auto issue = [&](int rb, int R1, int bb) {
    {  // 8 threads per row: row ri = tid / 8, 16-B chunks c = tid % 8 + 8 x (9 of q, 8 of dO)
      const int ri = tid >> 3, c0 = tid & 7;
      const bool v = rb + ri < R1;
      const int r = v ? rb + ri : 0, t = div_h(p, r), h = r - t * H;
      const uint16_t* qg = p.q + bi * p.q_sb + (int64_t)t * p.q_st + (int64_t)h * p.q_sh + 8 * c0;
      const uint16_t* og = p.dout + bi * p.o_sb + (int64_t)t * p.o_st + (int64_t)h * p.o_sh + 8 * c0;
      const uint32_t qs = sb + kKOffQ + (bb * kKRows + ri) * kQRow + 16 * c0;
      const uint32_t os = sb + kKOffDO + (bb * kKRows + ri) * kORow + 16 * c0;
#pragma unroll
      for (int u = 0; u < kDQK / 64; ++u) cp16(qs + 128 * u, qg + 64 * u, v);
#pragma unroll
      for (int u = 0; u < kDV / 64; ++u) cp16(os + 128 * u, og + 64 * u, v);
    }
    if (tid < kKRows) {
      const bool v = rb + tid < R1;
      const int r = v ? rb + tid : 0, t = div_h(p, r), h = r - t * H, pos = p.q_start + t;
      lse_s[bb * kKRows + tid] = v ? p.lse[((int64_t)bi * H + h) * p.n_q + t] * kLog2e : 0.f;
      D_s[bb * kKRows + tid] = v ? p.D[(int64_t)bi * rows + r] : 0.f;
      pos_s[bb * kKRows + tid] = v ? pos : -1;  // an invalid row attends nothing (j <= -1 fails; masked below)
      lb_s[bb * kKRows + tid] = pos / p.b - p.l + 1;
    }
    cp_commit();
  };
  // phase 1: warp (key half kh, k quarter kq) keeps its A fragments K[16 keys x 144 dims] in registers for the
  // CTA's lifetime (V = K[:, :512] reuses them) and computes partial S^T, dP^T over all 32 rows of a tile
  // (0.5 ldmatrix per MMA); the four quarters meet in shared memory. Phase 2: keys km, dims quarter qd.
  const int kh = warp & 1, kq = warp >> 1, km = 16 * kh, qd = kq;
  const int ndp = 32 - 9 * kq < 9 ? 32 - 9 * kq : 9;  // dP^T k steps of this quarter (dims < 512)
  // elementwise: thread -> key kk, rows 4 r4 .. + 3
  const int kk = tid >> 3, r4 = 4 * (tid & 7), jk = j0 + kk;
  const bool jokk = jk < p.n_kv, jsink = !p.sparse || kb < p.s;
  float* part = reinterpret_cast<float*>(smem + kKOffPart);
  float acc[34][4];
#pragma unroll
  for (int n = 0; n < 34; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.f;
  const uint32_t aK = sb + kKOffK + (km + (lane & 15)) * kQRow + (lane >> 4) * 16 + 32 * 9 * kq;
  // B of two 8-row n tiles x one k step (rows 16 np + .., k = 16 ks + ..)
  const uint32_t bQ = ((lane & 7) + ((lane >> 4) << 3)) * kQRow + ((lane >> 3) & 1) * 16 + 32 * 9 * kq;
  const uint32_t bO = ((lane & 7) + ((lane >> 4) << 3)) * kORow + ((lane >> 3) & 1) * 16 + 32 * 9 * kq;
  const uint32_t aP = sb + kKOffP + (km + (lane & 15)) * kTRow + (lane >> 4) * 16;
  const uint32_t aD = sb + kKOffDS + (km + (lane & 15)) * kTRow + (lane >> 4) * 16;
  const int trow = (lane & 7) + ((lane >> 3) & 1) * 8, tcol = (lane >> 4) * 8;  // ldmatrix.trans lane address
  int csig = -1, crb = 0, cre = 0;
  next_seg(csig, crb, cre);
  int nsig = csig, nrb = crb, nre = cre;
  if (csig < L) {
    issue(crb, cre, 0);
    advance(nsig, nrb, nre);
    cp_wait<1>();  // the K tile (committed first)
  } else {
    cp_wait<0>();
  }
  __syncthreads();
  uint32_t kfr[9][4];
#pragma unroll
  for (int i = 0; i < 9; ++i) ldsm4(aK + 32 * i, kfr[i]);
  for (int bb = 0; csig < L; bb ^= 1) {
    if (nsig < L) {
      issue(nrb, nre, bb ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const uint32_t qbase = sb + kKOffQ + bb * kKRows * kQRow, obase = sb + kKOffDO + bb * kKRows * kORow;
    float sp[4][4] = {}, dpp[4][4] = {};
#pragma unroll
    for (int i = 0; i < 9; ++i) {
#pragma unroll
      for (int np = 0; np < 2; ++np) {
        uint32_t b[4];
        ldsm4(qbase + bQ + 16 * np * kQRow + 32 * i, b);
        mma(sp[2 * np], kfr[i], b[0], b[1]);
        mma(sp[2 * np + 1], kfr[i], b[2], b[3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if (i < ndp) {
#pragma unroll
        for (int np = 0; np < 2; ++np) {
          uint32_t b[4];
          ldsm4(obase + bO + 16 * np * kORow + 32 * i, b);
          mma(dpp[2 * np], kfr[i], b[0], b[1]);
          mma(dpp[2 * np + 1], kfr[i], b[2], b[3]);
        }
      }
    }
    // partials: C fragment keys km + g (+8), rows 8 nt + 2 t4 (+1)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int off = (kq * kKKeys + km + g + 8 * u) * kPartRow + 8 * nt + 2 * t4;
        *reinterpret_cast<float2*>(part + off) = make_float2(sp[nt][2 * u], sp[nt][2 * u + 1]);
        *reinterpret_cast<float2*>(part + 4 * kKKeys * kPartRow + off) = make_float2(dpp[nt][2 * u], dpp[nt][2 * u + 1]);
      }
    __syncthreads();  // partials complete
    const int rb = crb, R1 = cre;
    float4 S4 = make_float4(0.f, 0.f, 0.f, 0.f), P4 = S4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 a = *reinterpret_cast<const float4*>(part + (q * kKKeys + kk) * kPartRow + r4);
      const float4 d = *reinterpret_cast<const float4*>(part + 4 * kKKeys * kPartRow + (q * kKKeys + kk) * kPartRow + r4);
      S4.x += a.x;
      S4.y += a.y;
      S4.z += a.z;
      S4.w += a.w;
      P4.x += d.x;
      P4.y += d.y;
      P4.z += d.z;
      P4.w += d.w;
    }
    const float sv[4] = {S4.x, S4.y, S4.z, S4.w}, dv4[4] = {P4.x, P4.y, P4.z, P4.w};
    float pv[4], dsv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int ri = r4 + e, r = rb + ri;
      // allowed(): causal j <= pos, then sink or inside the row's local window (invalid rows: pos = -1)
      const int pos = pos_s[bb * kKRows + ri];
      const bool ok = r < R1 && jokk && (!p.causal || jk <= pos) && (jsink || kb >= lb_s[bb * kKRows + ri]);
      pv[e] = ok ? ex2f(fmaf(sv[e], p.sl2, -lse_s[bb * kKRows + ri])) : 0.f;
      dsv[e] = pv[e] * (dv4[e] - D_s[bb * kKRows + ri]);
    }
    {
      const uint32_t off = kk * kTRow + r4 * 2;
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(sb + kKOffP + off), "r"(pack2(pv[0], pv[1])),
                   "r"(pack2(pv[2], pv[3])));
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(sb + kKOffDS + off), "r"(pack2(dsv[0], dsv[1])),
                   "r"(pack2(dsv[2], dsv[3])));
    }
    __syncthreads();  // P^T, dS^T complete
    uint32_t ad0[4], ad1[4], ap0[4], ap1[4];
    ldsm4(aD, ad0);
    ldsm4(aD + 32, ad1);
    ldsm4(aP, ap0);
    ldsm4(aP + 32, ap1);
#pragma unroll
    for (int np = 0; np < 17; ++np) {
      const int n0 = 34 * qd + 2 * np;  // first of this pair of 8-wide n tiles in [dK | dV]
      uint32_t b[4];
      if (n0 < kDQK / 8) {
        const uint32_t base = qbase + trow * kQRow + (8 * n0 + tcol) * 2;
        ldsm4t(base, b);
        mma(acc[2 * np], ad0, b[0], b[1]);
        mma(acc[2 * np + 1], ad0, b[2], b[3]);
        ldsm4t(base + 16 * kQRow, b);
        mma(acc[2 * np], ad1, b[0], b[1]);
        mma(acc[2 * np + 1], ad1, b[2], b[3]);
      } else {
        const uint32_t base = obase + trow * kORow + (8 * n0 - kDQK + tcol) * 2;
        ldsm4t(base, b);
        mma(acc[2 * np], ap0, b[0], b[1]);
        mma(acc[2 * np + 1], ap0, b[2], b[3]);
        ldsm4t(base + 16 * kORow, b);
        mma(acc[2 * np], ap1, b[0], b[1]);
        mma(acc[2 * np + 1], ap1, b[2], b[3]);
      }
    }
    __syncthreads();  // buffers bb and the P / dS tiles free
    csig = nsig;
    crb = nrb;
    cre = nre;
    if (nsig < L) advance(nsig, nrb, nre);
  }
  cp_wait<0>();  // (no row tiles: the K tile copy)
  // C fragment: keys km + g (+8), columns 8 n + 2 t4 of [dK | dV]
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int kl = km + g + 8 * u, j = j0 + kl;
    if (j >= p.n_kv) continue;
    if (split) {
      float* out = p.part + ((((int64_t)bi * p.n_sink + tile) * p.nsplit + blockIdx.y) * kKKeys + kl) * kDKV;
#pragma unroll
      for (int np = 0; np < 34; ++np) {
        const int c = 8 * (34 * qd + np) + 2 * t4;
        const float sc = c < kDQK ? p.scale : 1.f;
        *reinterpret_cast<float2*>(out + c) = make_float2(acc[np][2 * u] * sc, acc[np][2 * u + 1] * sc);
      }
    } else {
#pragma unroll
      for (int np = 0; np < 34; ++np) {
        const int c = 8 * (34 * qd + np) + 2 * t4;
        if (c < kDQK)
          *reinterpret_cast<float2*>(p.dk + ((int64_t)bi * p.n_kv + j) * kDQK + c) =
              make_float2(acc[np][2 * u] * p.scale, acc[np][2 * u + 1] * p.scale);
        else
          *reinterpret_cast<float2*>(p.dv + ((int64_t)bi * p.n_kv + j) * kDV + c - kDQK) =
              make_float2(acc[np][2 * u], acc[np][2 * u + 1]);
      }
    }
  }
}

// sink-tile partials -> dK / dV, summed over the splits in a fixed order
__global__ void __launch_bounds__(256) bwd_sink_reduce_kernel(MP p) {
  const int64_t per = (int64_t)p.n_sink * kKKeys * (kDKV / 4);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)p.batch * per) return;
  const int bi = (int)(i / per);
  const int64_t rem = i - bi * per;
  const int tile = (int)(rem / (kKKeys * (kDKV / 4)));
  const int r2 = (int)(rem - (int64_t)tile * kKKeys * (kDKV / 4));
  const int kl = r2 / (kDKV / 4), c = 4 * (r2 - kl * (kDKV / 4));
  const int j = tile * kKKeys + kl;
  if (j >= p.n_kv) return;
  const float* src = p.part + (((int64_t)bi * p.n_sink + tile) * p.nsplit * kKKeys + kl) * kDKV + c;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int y = 0; y < p.nsplit; ++y) {
    const float4 v = *reinterpret_cast<const float4*>(src + (int64_t)y * kKKeys * kDKV);
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  float* dst = c < kDQK ? p.dk + ((int64_t)bi * p.n_kv + j) * kDQK + c : p.dv + ((int64_t)bi * p.n_kv + j) * kDV + c - kDQK;
  *reinterpret_cast<float4*>(dst) = s;
}

int sink_splits(const AttnProblem& a) {
  if (!a.sparse || a.s == 0 || a.n_kv == 0) return 1;  // no sink tiles: nothing to split
  if (backward_pair_eligible(a)) return backward_pair_splits(a).nsplit;  // pieces as long as the local tiles' 
  const int64_t win = (int64_t)a.l * a.b;
  int64_t n = (a.n_q + win - 1) / win;
  return (int)(n < 1 ? 1 : n > 64 ? 64 : n);
}
int sink_tiles(const AttnProblem& a) {
  const int64_t se = (int64_t)a.s * a.b < a.n_kv ? (int64_t)a.s * a.b : a.n_kv;
  return (int)((se + kKKeys - 1) / kKKeys);
}

}  // namespace

// per-device side stream + fork / join events of the backward (D beside the dV kernel); per host thread
struct SideCtx {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
cudaError_t side_ctx(SideCtx** out) {
  static thread_local SideCtx ctx[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  SideCtx& c = ctx[dev];
  if (!c.side) {
    e = cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      c.side = nullptr;
      return e;
    }
  }
  *out = &c;
  return cudaSuccess;
}

size_t backward_mma_part_bytes(const AttnProblem& a) {
  if (!a.sparse || sink_splits(a) <= 1) return 0;
  return sizeof(float) * (size_t)a.batch * sink_tiles(a) * sink_splits(a) * kKKeys * kDKV;
}

bool backward_mma_eligible(const AttnProblem& a, const void* dout) {
  const auto& kv = a.kv.seg[0];
  auto al = [](const void* x) { return (reinterpret_cast<uintptr_t>(x) & 15) == 0; };
  const bool v_alias = kv.v == kv.k && kv.v_st == kv.k_st && kv.v_sb == kv.k_sb;
  return a.in_bf16 && a.out_bf16 && a.d_qk == kDQK && a.d_v == kDV && v_alias && (!a.sparse || a.b % kKKeys == 0) &&
         al(a.q) && al(kv.k) && al(a.o) && al(dout) && a.q_sb % 8 == 0 && a.q_st % 8 == 0 && a.q_sh % 8 == 0 &&
         kv.k_sb % 8 == 0 && kv.k_st % 8 == 0 && a.o_sb % 8 == 0 && a.o_st % 8 == 0 && a.o_sh % 8 == 0 &&
         a.n_kv + a.q_start < (int64_t)1 << 30 && (int64_t)a.n_q * a.heads < (int64_t)1 << 30;
}

cudaError_t launch_attn_backward_mma(const AttnProblem& a, const void* dout, float* dq, float* dk, float* dv,
                                     float* D, float* part, uint16_t* ds, cudaStream_t st) {
  MP p;
  const auto& kv = a.kv.seg[0];
  p.q = static_cast<const uint16_t*>(a.q);
  p.k = static_cast<const uint16_t*>(kv.k);
  p.o = static_cast<const uint16_t*>(a.o);
  p.dout = static_cast<const uint16_t*>(dout);
  p.lse = a.lse;
  p.dq = dq;
  p.dk = dk;
  p.dv = dv;
  p.D = D;
  p.part = part;
  p.q_sb = a.q_sb;
  p.q_st = a.q_st;
  p.q_sh = a.q_sh;
  p.k_sb = kv.k_sb;
  p.k_st = kv.k_st;
  p.o_sb = a.o_sb;
  p.o_st = a.o_st;
  p.o_sh = a.o_sh;
  p.batch = a.batch;
  p.n_q = a.n_q;
  p.heads = a.heads;
  p.n_kv = (int32_t)a.n_kv;
  p.q_start = (int32_t)a.q_start;
  p.scale = a.scale;
  p.sl2 = a.scale * kLog2e;
  p.sparse = a.sparse;
  p.causal = a.causal;
  p.s = a.s;
  p.l = a.l;
  p.b = a.b;
  p.nsplit = sink_splits(a);
  p.n_sink = sink_tiles(a);
  fastdiv_init((uint32_t)a.heads, p.h_m, p.h_p);
  const bool use_part = a.sparse && p.nsplit > 1;
  if (use_part && !part) return cudaErrorInvalidValue;
  const int64_t rows = (int64_t)a.n_q * a.heads;
  cudaError_t e;
  // Key side: tcgen05 (attn_bwd_tc.cu) for the packed row layout (test knob backward = 2 forces this file's key
  // kernel). SSA: the tcgen05 key kernel also writes dS rows and dQ = dS K runs as a tcgen05 GEMM
  // (knob backward = 3 keeps this file's row kernel, which recomputes S and dP).
  const bool force_mma = knob(kKnobBackward) == 2;
  const bool force_dq_mma = knob(kKnobBackward) == 3;
  const bool tc_keys = !force_mma && backward_tc_eligible(a, dout);
  // 64-key tiles (a dV kernel and a dK kernel, attn_bwd_tc.cu; 128-key CTA-pair kernels for SSA with b = 128
  // unless the test knob backward = 5) unless the tile would straddle a block or the test knob backward = 4
  // keeps the 32-key kernel that accumulates dK and dV in one pass
  const bool key64 = knob(kKnobBackward) != 4 && backward_key64_eligible(a);
  if (tc_keys && !force_dq_mma && ds && backward_ds_eligible(a) && rows > 0 && a.n_kv > 0) {
    if (key64) {
      // D = rowsum(dO O) on a side stream, beside the dV kernel (which does not read it; its CTAs leave room
      // for D's), joined before the dK kernel
      SideCtx* sc = nullptr;
      if ((e = side_ctx(&sc)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(sc->fork, st)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(sc->side, sc->fork, 0)) != cudaSuccess) return e;
      if ((e = launch_bwd_D(a, dout, D, sc->side)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(sc->join, sc->side)) != cudaSuccess) return e;
      // the local-tile row-split partials follow the sink partials in the workspace
      float* part_local = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(part) +
                                                   (backward_mma_part_bytes(a) + 255) / 256 * 256);
      e = launch_bwd_key64_tc(a, dout, dk, dv, D, part, ds, p.nsplit, p.n_sink, st, sc->join,
                              knob(kKnobBackward) != 5, part_local);
    } else {
      if ((e = launch_bwd_D(a, dout, D, st)) != cudaSuccess) return e;
      e = launch_bwd_dkdv_tc(a, dout, dk, dv, D, part, ds, p.nsplit, p.n_sink, st);
    }
    if (e != cudaSuccess) return e;
    const bool pair_keys = key64 && knob(kKnobBackward) != 5 && backward_pair_eligible(a);
    if ((e = launch_bwd_dq_tc(a, ds, dq, st, pair_keys)) != cudaSuccess) return e;
    if (use_part) {
      const int64_t n = (int64_t)a.batch * p.n_sink * kKKeys * (kDKV / 4);
      bwd_sink_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p);
      count_launch();
    }
    return cudaGetLastError();
  }
  if (rows > 0) {
    e = cudaFuncSetAttribute(bwd_dq_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRSmem);
    if (e != cudaSuccess) return e;
    const int64_t rt = (rows + kRRows - 1) / kRRows;
    bwd_dq_mma_kernel<<<(unsigned)(a.batch * rt), 256, kRSmem, st>>>(p);
    count_launch();
  }
  if (a.n_kv > 0) {
    if (tc_keys) {
      e = key64 ? launch_bwd_key64_tc(a, dout, dk, dv, D, part, nullptr, p.nsplit, p.n_sink, st)
                : launch_bwd_dkdv_tc(a, dout, dk, dv, D, part, nullptr, p.nsplit, p.n_sink, st);
      if (e != cudaSuccess) return e;
    } else {
      e = cudaFuncSetAttribute(bwd_dkdv_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kKSmem);
      if (e != cudaSuccess) return e;
      const int64_t kt = (a.n_kv + kKKeys - 1) / kKKeys;
      bwd_dkdv_mma_kernel<<<dim3((unsigned)(a.batch * kt), use_part ? p.nsplit : 1), 256, kKSmem, st>>>(p);
      count_launch();
    }
    if (use_part) {
      const int64_t n = (int64_t)a.batch * p.n_sink * kKKeys * (kDKV / 4);
      bwd_sink_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p);
      count_launch();
    }
  }
  return cudaGetLastError();
}

}  // namespace loza
