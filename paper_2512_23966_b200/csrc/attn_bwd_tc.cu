// Attention backward, key side on the 5th-gen tensor cores: dK_j = scale sum_r dS_rj q_r and
// dV_j = sum_r P_rj dO_r (definitions in attn_bwd_simt.cu's header) for the absorbed MLA shape (bf16, d_qk 576,
// d_v 512, V = K[:, :512]) with tcgen05 UMMAs, fp32 accumulators in TMEM. The dQ / D side stays on the row
// kernel of attn_bwd_mma.cu (launched first: D feeds this kernel).
//
// One CTA per 32 keys of one b-block (the key tile of attn_bwd_mma.cu's key kernel, same row ranges, sink
// splits and row-block rotation), rows streamed as 128-row tiles:
//   S   [128 rows x 32 keys] = Q K^T        (A = Q K-major, B = K K-major; M128 N32, 36 k steps)
//   dP  [128 x 32]           = dO V^T       (32 k steps)
//   P, dS = f(S, dP) by 4 warps (thread = row = TMEM lane), bf16 into shared memory ([rows][32 keys], SW64)
//   dK^T [576 x 32] += Q^T dS                (A = Q^T MN-major from the same SW128 boxes; 5 M128 tiles, the
//                                             last over dims 512..639 whose upper half TMA zero-fills)
//   dV^T [512 x 32] += dO^T P                (4 M128 tiles)
// TMEM: dK^T 160 + dV^T 128 + S 2x32 + dP 2x32 columns. Q / dO move as 64-dim chunk pairs [2][128 rows][64]
// (one 4-D TMA box, 32 KB) through a 5-slot ring, twice per row tile (S/dP, then dK^T/dV^T): the tile does
// not fit shared memory whole. Warp roles: 0 TMA, 1 UMMA issue (+ TMEM alloc), 4-7 P/dS and the epilogue.
#include <math.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {

using namespace sm100;

constexpr int kKeys = 32, kRows = 128, kDqk = 576, kDv = 512, kDkv = kDqk + kDv;
constexpr int kQPairs = 5, kOPairs = 4;        // 64-dim chunk pairs of q (the 10th chunk is OOB: zeros) and dO
constexpr int kPairBytes = 2 * kRows * 128;    // 32 KB
constexpr int kStages = 5;
constexpr int kPBufs = 1;  // P/dS buffers (one: the shared memory goes to a 5th ring slot)
constexpr int kKBytes = 9 * kKeys * 128;       // 36 KB: [9 chunks][32 keys][64]
constexpr int kPBytes = kRows * 64;            // [128 rows][32 keys] bf16, SWIZZLE_64B
constexpr int kOffRing = 0;
constexpr int kOffK = kOffRing + kStages * kPairBytes;
constexpr int kOffP = kOffK + kKBytes;         // kPBufs buffers each for P and dS
constexpr int kOffDS = kOffP + kPBufs * kPBytes;
constexpr int kOffBar = kOffDS + kPBufs * kPBytes;
constexpr int kBarFull = 0, kBarEmpty = kStages, kBarK = 2 * kStages, kBarSFull = kBarK + 1,
              kBarSFree = kBarSFull + 2, kBarPReady = kBarSFree + 2, kBarPFree = kBarPReady + 2,
              kBarAcc = kBarPFree + 2, kNumBars = kBarAcc + 1;
constexpr int kOffTmemPtr = kOffBar + 8 * kNumBars;
constexpr int kSmem = kOffTmemPtr + 16 + 1024;  // + alignment slack (SW128 operands: 1024-B aligned)
constexpr uint32_t kTmemDK = 0, kTmemDV = 160, kTmemS = 288, kTmemDP = 352, kTmemCols = 512;
constexpr float kLog2e = 1.4426950408889634f;

struct TcBwdParams {
  CUtensorMap q_map;  // {64, n_q*H rows, 9 chunks, B}, box {64, 128, 2, 1}
  CUtensorMap o_map;  // dO: {64, n_q*H, 8, B}, box {64, 128, 2, 1}
  CUtensorMap k_map;  // {64, n_kv, 9, B}, box {64, 32, 9, 1}
  CUtensorMap q4_map, q1_map, o4_map;  // pair kernels: q / dO boxes {64, 64, 4 (q1: 1), 1}
  CUtensorMap ds_map;                  // pair kernels: the dS row buffer {W slots, n_q*H rows, B}, box {64, 128, 1}
  const float* lse;
  const float* D;
  float* dk;
  float* dv;
  float* part;
  float* part_local;  // pair kernels with local row splits: [B][kt - ns][lsplit][128][1088]
  uint16_t* ds;  // SSA: dS rows [B][n_q*H][(s+l)*b] bf16 (slot = sink key, then the row's local window), or NULL
  int32_t batch, n_q, heads, n_kv, q_start;
  float scale, sl2;
  int32_t sparse, causal, s, l, b;
  int32_t nsplit, n_sink;
  int32_t lsplit;  // pair kernels: row splits of every local tile (1: none)
  uint32_t h_m, h_p;
  unsigned long long* trace;  // debug timeline of pair cluster trace_cluster (pair kernels; NULL in production)
  int32_t trace_cluster;
};

__device__ __forceinline__ int div_h(const TcBwdParams& p, int n) {
  return (int)(((uint64_t)(uint32_t)n * p.h_m) >> p.h_p);
}
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;  // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ void st_shared_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// The CTA's row tiles (all roles walk the same sequence): segments as in attn_bwd_mma.cu's key kernel.
struct RowIter {
  int L, m0, m1, p0, p1, R0, R1, qs, H, b;
  int step = kRows;  // rows per tile
  int sig, m, rb, re;
  // L == 1: the row range [R0, R1) in order. L > 1: the query blocks m0 .. m1 in the order (m mod L, m), so at
  // step sig every CTA of the grid streams blocks m = sig (mod L) and the CTAs that share a block read it together
  __device__ void next_seg() {
    for (;;) {
      if (L == 1) {
        if (++sig >= 1) return;
        rb = R0;
        re = R1;
      } else {
        m += L;
        if (sig < 0 || m > m1) {
          if (++sig >= L) return;
          m = m0 + ((sig - m0) % L + L) % L;
          if (m > m1) continue;
        }
        const int a = m * b > p0 ? m * b : p0, e = (m + 1) * b < p1 ? (m + 1) * b : p1;
        rb = (a - qs) * H;
        re = (e - qs) * H;
      }
      if (rb < re) return;
    }
  }
  __device__ void start() {
    sig = -1;
    m = 0;
    rb = re = 0;
    next_seg();
  }
  __device__ bool valid() const { return sig < L; }
  __device__ void advance() {
    rb += step;
    if (rb >= re) next_seg();
  }
};

__global__ void __launch_bounds__(256, 1) bwd_dkdv_tc_kernel(const __grid_constant__ TcBwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sbase - sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = p.heads;
  const int ktiles = (p.n_kv + kKeys - 1) / kKeys;
  // blocks of a batch entry: the sink tiles' row splits first (as long as a full local tile: they must not
  // start late), then one per local tile
  const int nst = p.sparse && p.nsplit > 1 ? (int)(((int64_t)p.s * p.b + kKeys - 1) / kKeys) : 0;
  const int ns = nst < ktiles ? nst : ktiles;
  const int units = ns * p.nsplit + (ktiles - ns);
  const int bi = (int)blockIdx.x / units, u = (int)blockIdx.x - bi * units;
  const int tile = u < ns * p.nsplit ? u / p.nsplit : ns + (u - ns * p.nsplit);
  const int ys = u < ns * p.nsplit ? u - tile * p.nsplit : 0;  // row split of a sink tile
  const int j0 = tile * kKeys;
  // rows attending keys [j0, j0 + 32): positions [p0, p1) (as in attn_bwd_mma.cu)
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
    // a sink tile's rows split by whole query blocks, each split walked in the local tiles' rotation (its reads
    // hit the rows the local tiles stream at the same step)
    if (p1 > p0) {
      const int ma = p0 / p.b, nb = (p1 - 1) / p.b - ma + 1, cb = (nb + p.nsplit - 1) / p.nsplit;
      const int a = (ma + ys * cb) * p.b, e = a + cb * p.b;
      if (a > p0) p0 = a;
      if (e < p1) p1 = e;
    }
    R0 = R1 = 0;
    if (p1 > p0) {
      R0 = (p0 - p.q_start) * H;
      R1 = (p1 - p.q_start) * H;
    }
  }
  RowIter it;
  it.L = p.sparse && (split || kb >= p.s) ? p.l : 1;
  it.m0 = p0 / p.b;
  it.m1 = (p1 - 1) / p.b;
  it.p0 = p0;
  it.p1 = p1;
  it.R0 = R0;
  it.R1 = R1;
  it.qs = p.q_start;
  it.H = H;
  it.b = p.b;
  it.start();
  const bool any = it.valid();

  auto bar = [&](int i) { return sbase + kOffBar + 8 * i; };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar(kBarFull + i), 1);
      mbar_init(bar(kBarEmpty + i), 1);
    }
    mbar_init(bar(kBarK), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), 4);
      mbar_init(bar(kBarPReady + i), 4);
      mbar_init(bar(kBarPFree + i), 1);
    }
    mbar_init(bar(kBarAcc), 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.o_map);
    prefetch_tmap(&p.k_map);
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_ptr), kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0 && any) {
      const uint64_t pol_k = policy_evict_last(), pol = policy_evict_normal();
      mbar_arrive_expect_tx(bar(kBarK), kKBytes);
      tma_load_4d(sbase + kOffK, &p.k_map, 0, j0, 0, bi, bar(kBarK), pol_k);
      uint32_t slot = 0, ph = 0;
      auto load_pair = [&](const CUtensorMap* m, int pair, int rb) {
        mbar_wait(bar(kBarEmpty + slot), ph ^ 1);
        mbar_arrive_expect_tx(bar(kBarFull + slot), kPairBytes);
        tma_load_4d(sbase + kOffRing + slot * kPairBytes, m, 0, rb, 2 * pair, bi, bar(kBarFull + slot), pol);
        if (++slot == kStages) {
          slot = 0;
          ph ^= 1;
        }
      };
      // the UMMA issuer's order: S/dP of tile t + 1 before dK^T/dV^T of tile t
      auto load_tile = [&](int rb) {
        for (int q = 0; q < kQPairs; ++q) load_pair(&p.q_map, q, rb);
        for (int q = 0; q < kOPairs; ++q) load_pair(&p.o_map, q, rb);
      };
      RowIter ia = it;
      load_tile(ia.rb);
      ia.advance();
      for (; it.valid(); it.advance()) {
        if (ia.valid()) {
          load_tile(ia.rb);
          ia.advance();
        }
        load_tile(it.rb);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ UMMA issuer
    if (any) {
      constexpr uint32_t id_s = idesc_bf16_f32(kRows, kKeys, false, false);
      constexpr uint32_t id_t = idesc_bf16_f32(128, kKeys, true, true);
      mbar_wait(bar(kBarK), 0);
      tc_fence_after();
      uint32_t slot = 0, ph = 0;
      auto take = [&]() {
        mbar_wait(bar(kBarFull + slot), ph);
        tc_fence_after();
      };
      auto release = [&]() {
        if (elect_one()) umma_commit_1sm(bar(kBarEmpty + slot));
        __syncwarp();
        if (++slot == kStages) {
          slot = 0;
          ph ^= 1;
        }
      };
      // S/dP of tile t + 1 are issued before dK^T/dV^T of tile t (S/dP double-buffered in TMEM), so the
      // tensor pipe works while the four P/dS warps process tile t
      auto issue_sdp = [&](int tc) {
        const int buf = tc & 1, use = tc >> 1;
        mbar_wait(bar(kBarSFree + buf), (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t tS = tmem + kTmemS + 32 * buf, tP = tmem + kTmemDP + 32 * buf;
        for (int q = 0; q < kQPairs; ++q) {  // S = Q K^T
          take();
          if (elect_one()) {
            const int nk = q < kQPairs - 1 ? 8 : 4;
            for (int k = 0; k < nk; ++k) {
              const uint32_t ch = 2 * q + (k >> 2), kk = k & 3;
              umma_bf16_1sm(tS, sdesc_sw128(sbase + kOffRing + slot * kPairBytes + (k >> 2) * 16384 + 32 * kk, 16, 1024),
                            sdesc_sw128(sbase + kOffK + ch * 4096 + 32 * kk, 16, 1024), id_s, (q | k) != 0);
            }
          }
          release();
        }
        for (int q = 0; q < kOPairs; ++q) {  // dP = dO V^T (V = K[:, :512])
          take();
          if (elect_one()) {
            for (int k = 0; k < 8; ++k) {
              const uint32_t ch = 2 * q + (k >> 2), kk = k & 3;
              umma_bf16_1sm(tP, sdesc_sw128(sbase + kOffRing + slot * kPairBytes + (k >> 2) * 16384 + 32 * kk, 16, 1024),
                            sdesc_sw128(sbase + kOffK + ch * 4096 + 32 * kk, 16, 1024), id_s, (q | k) != 0);
            }
          }
          release();
        }
        if (elect_one()) umma_commit_1sm(bar(kBarSFull + buf));
        __syncwarp();
      };
      auto issue_grad = [&](int tc) {
        const int buf = tc % kPBufs, use = tc / kPBufs;
        mbar_wait(bar(kBarPReady + buf), use & 1);
        tc_fence_after();
        const uint32_t dsb = sbase + kOffDS + buf * kPBytes, pb = sbase + kOffP + buf * kPBytes;
        for (int q = 0; q < kQPairs; ++q) {  // dK^T[dims 128 q ..] += Q^T dS
          take();
          if (elect_one()) {
            for (int kr = 0; kr < 8; ++kr)
              umma_bf16_1sm(tmem + kTmemDK + 32 * q,
                            sdesc_sw128(sbase + kOffRing + slot * kPairBytes + 2048 * kr, 16384, 1024),
                            sdesc_sw64(dsb + 1024 * kr, 16, 512), id_t, (tc | kr) != 0);
          }
          release();
        }
        for (int q = 0; q < kOPairs; ++q) {  // dV^T[dims 128 q ..] += dO^T P
          take();
          if (elect_one()) {
            for (int kr = 0; kr < 8; ++kr)
              umma_bf16_1sm(tmem + kTmemDV + 32 * q,
                            sdesc_sw128(sbase + kOffRing + slot * kPairBytes + 2048 * kr, 16384, 1024),
                            sdesc_sw64(pb + 1024 * kr, 16, 512), id_t, (tc | kr) != 0);
          }
          release();
        }
        if (elect_one()) umma_commit_1sm(bar(kBarPFree + buf));
        __syncwarp();
      };
      RowIter ia = it;
      issue_sdp(0);
      ia.advance();
      int ta = 1;
      for (int tc = 0; it.valid(); it.advance(), ++tc) {
        if (ia.valid()) {
          issue_sdp(ta++);
          ia.advance();
        }
        issue_grad(tc);
      }
      if (elect_one()) umma_commit_1sm(bar(kBarAcc));
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ P / dS (thread = row = TMEM lane)
    const int q = warp - 4, row = 32 * q + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const int rows = p.n_q * H;
    const bool jsink = !p.sparse || kb < p.s;
    for (int tc = 0; it.valid(); it.advance(), ++tc) {
      const int buf = tc & 1, use = tc >> 1;
      const int r = it.rb + row;
      const bool rv = r < it.re;
      const int rr = rv ? r : 0, t = div_h(p, rr), h = rr - t * H, pos = p.q_start + t;
      const float lse2 = rv ? p.lse[((int64_t)bi * H + h) * p.n_q + t] * kLog2e : 0.f;
      const float Dr = rv ? p.D[(int64_t)bi * rows + rr] : 0.f;
      const bool win = jsink || kb >= pos / p.b - p.l + 1;
      mbar_wait(bar(kBarSFull + buf), use & 1);
      tc_fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld32(tl + kTmemS + 32 * buf, sv);
      tmem_ld32(tl + kTmemDP + 32 * buf, dv);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarSFree + buf));
      uint32_t pk[16], dk2[16];
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        float pv[2], ds[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = j0 + c + e;
          const bool ok = rv && win && j < p.n_kv && (!p.causal || j <= pos);
          pv[e] = ok ? ex2(fmaf(__uint_as_float(sv[c + e]), p.sl2, -lse2)) : 0.f;
          ds[e] = pv[e] * (__uint_as_float(dv[c + e]) - Dr);
        }
        pk[c >> 1] = pack_bf16x2(pv[0], pv[1]);
        dk2[c >> 1] = pack_bf16x2(ds[0], ds[1]);
      }
      if (p.ds && rv) {  // this row's 32 dS values at its slots of block kb (every row here has kb in its window)
        int lbq = pos / p.b - p.l + 1;
        if (lbq < p.s) lbq = p.s;
        const int W = (p.s + p.l) * p.b;
        const int slot = kb < p.s ? j0 : p.s * p.b + (kb - lbq) * p.b + (j0 - kb * p.b);
        uint4* dst = reinterpret_cast<uint4*>(p.ds + ((int64_t)bi * rows + rr) * W + slot);
#pragma unroll
        for (int u = 0; u < 4; ++u) dst[u] = make_uint4(dk2[4 * u], dk2[4 * u + 1], dk2[4 * u + 2], dk2[4 * u + 3]);
      }
      const int pbuf = tc % kPBufs, puse = tc / kPBufs;
      mbar_wait(bar(kBarPFree + pbuf), (puse & 1) ^ 1);
      // row of 64 B = 4 x 16-B units, SWIZZLE_64B: unit u at (u ^ (row >> 1) & 3)
      const uint32_t pr = sbase + kOffP + pbuf * kPBytes + row * 64, dr = sbase + kOffDS + pbuf * kPBytes + row * 64;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t o = (uint32_t)((u ^ ((row >> 1) & 3)) << 4);
        st_shared_v4(pr + o, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        st_shared_v4(dr + o, dk2[4 * u], dk2[4 * u + 1], dk2[4 * u + 2], dk2[4 * u + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarPReady + pbuf));
    }
    // ------------------------------------------------------------------ epilogue: TMEM lane = dim, column = key
    if (any) {
      mbar_wait(bar(kBarAcc), 0);
      tc_fence_after();
    }
    for (int m = 0; m < kQPairs + kOPairs; ++m) {
      const bool isk = m < kQPairs;
      const int dim = 128 * (isk ? m : m - kQPairs) + 32 * q + lane;
      if (isk && 128 * m + 32 * q >= kDqk) continue;  // warp-uniform: dims 576.. of the last dK^T tile
      uint32_t v[32];
      if (any) {
        tmem_ld32(tl + (isk ? kTmemDK + 32 * m : kTmemDV + 32 * (m - kQPairs)), v);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = 0u;
      }
      const float sc = isk ? p.scale : 1.f;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int j = j0 + c;
        if (j >= p.n_kv) continue;
        const float x = __uint_as_float(v[c]) * sc;
        if (split)
          p.part[((((int64_t)bi * p.n_sink + tile) * p.nsplit + ys) * kKeys + c) * kDkv + (isk ? 0 : kDqk) + dim] = x;
        else if (isk)
          p.dk[((int64_t)bi * p.n_kv + j) * kDqk + dim] = x;
        else
          p.dv[((int64_t)bi * p.n_kv + j) * kDv + dim] = x;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, kTmemCols);
  }
}

// ------------------------------------------------------------------------------ key side, 64-key tiles
// The 32-key kernel above holds dK^T and dV^T of its keys in TMEM (288 columns) and so streams every row tile
// past 32 keys, twice. Here the key side is split into two kernels over 64-key tiles, each with one
// accumulator (MODE kDvOnly: dV^T = dO^T P, 4 x 64 columns; MODE kDkOnly: dK^T = Q^T dS, 5 x 64 columns):
//   dV kernel: S = Q K^T (Q pairs once), P = exp2(S scale log2e - LSE log2e), dV^T += dO^T P (dO pairs once)
//   dK kernel: S = Q K^T, dP = dO V^T (Q, dO pairs), dS = P (dP - D), dK^T += Q^T dS (Q pairs again); it also
//              writes the dS rows the dQ GEMM reads.
// Per 128-row tile and 64 keys the two kernels move Q 3x + dO 2x (703 KB) where the 32-key kernel moves
// Q 4x + dO 4x (1112 KB), and every UMMA is M128 N64 (48 tensor cycles) instead of M128 N32.
// TMEM: dV kernel dV^T 256 + S 2 x 64; dK kernel dK^T 320 + S 64 + dP 64 (single-buffered: the P/dS warps
// release them right after their TMEM loads). SMEM: ring 4 x 32 KB, K tile 72 KB, P or dS 16 KB (SW128).
constexpr int kDvOnly = 1, kDkOnly = 2, kDkFromP = 3;
constexpr int k64Keys = 64;
constexpr int k64Stages = 4;
constexpr int k64KBytes = 9 * k64Keys * 128;       // 72 KB: [9 chunks][64 keys][64]
constexpr int k64PBytes = kRows * 128;             // [128 rows][64 keys] bf16, SWIZZLE_128B
constexpr int k64OffRing = 0;
constexpr int k64OffK = k64OffRing + k64Stages * kPairBytes;
constexpr int k64OffP = k64OffK + k64KBytes;
constexpr int k64OffBar = k64OffP + k64PBytes;
constexpr int k64BarFull = 0, k64BarEmpty = k64Stages, k64BarK = 2 * k64Stages, k64BarSFull = k64BarK + 1,
              k64BarSFree = k64BarSFull + 2, k64BarPReady = k64BarSFree + 2, k64BarPFree = k64BarPReady + 1,
              k64BarAcc = k64BarPFree + 1, k64NumBars = k64BarAcc + 1;
constexpr int k64OffTmemPtr = k64OffBar + 8 * k64NumBars;
constexpr int k64Smem = k64OffTmemPtr + 16 + 1024;
static_assert(k64Smem <= 232448, "smem");

// MODE kDkFromP (SSA, with the dS row buffer): the dV kernel has left P (bf16) in the dS rows' slots, so the dK
// kernel reads P there instead of recomputing S: its first pass is dP = dO V^T only (dP double-buffered in
// TMEM), and it overwrites each slot with dS = P (dP - D). Per 128-row tile it moves dO + Q + 16 KB of P.
template <int MODE>
__global__ void __launch_bounds__(256, 1) bwd_key64_tc_kernel(const __grid_constant__ TcBwdParams p) {
  constexpr bool kIsDv = MODE == kDvOnly;
  constexpr bool kFromP = MODE == kDkFromP;
  constexpr int kSBufs = kIsDv || kFromP ? 2 : 1;  // S (and / or dP) buffers in TMEM
  constexpr uint32_t kTmemAcc = 0;                  // dV^T: 4 x 64 columns, dK^T: 5 x 64
  constexpr uint32_t kTmemS = kIsDv ? 256 : 320, kTmemDP = kFromP ? 320 : 384;
  constexpr uint32_t kDPStride = kFromP ? 64 : 0;   // dP buffer stride (double-buffered when S is not computed)
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sbase - sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int H = p.heads;
  const int ktiles = (p.n_kv + k64Keys - 1) / k64Keys;
  // blocks of a batch entry: the sink tiles' row splits first (as long as a full local tile: they must not
  // start late), then one per local tile
  const int nst = p.sparse && p.nsplit > 1 ? (int)(((int64_t)p.s * p.b + k64Keys - 1) / k64Keys) : 0;
  const int ns = nst < ktiles ? nst : ktiles;
  const int units = ns * p.nsplit + (ktiles - ns);
  const int bi = (int)blockIdx.x / units, u = (int)blockIdx.x - bi * units;
  const int tile = u < ns * p.nsplit ? u / p.nsplit : ns + (u - ns * p.nsplit);
  const int ys = u < ns * p.nsplit ? u - tile * p.nsplit : 0;  // row split of a sink tile
  const int j0 = tile * k64Keys;
  // rows attending keys [j0, j0 + 64) (b % 64 == 0: the tile lies in one block)
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
    // a sink tile's rows split by whole query blocks, each split walked in the local tiles' rotation (its reads
    // hit the rows the local tiles stream at the same step)
    if (p1 > p0) {
      const int ma = p0 / p.b, nb = (p1 - 1) / p.b - ma + 1, cb = (nb + p.nsplit - 1) / p.nsplit;
      const int a = (ma + ys * cb) * p.b, e = a + cb * p.b;
      if (a > p0) p0 = a;
      if (e < p1) p1 = e;
    }
    R0 = R1 = 0;
    if (p1 > p0) {
      R0 = (p0 - p.q_start) * H;
      R1 = (p1 - p.q_start) * H;
    }
  }
  RowIter it;
  it.L = p.sparse && (split || kb >= p.s) ? p.l : 1;
  it.m0 = p0 / p.b;
  it.m1 = (p1 - 1) / p.b;
  it.p0 = p0;
  it.p1 = p1;
  it.R0 = R0;
  it.R1 = R1;
  it.qs = p.q_start;
  it.H = H;
  it.b = p.b;
  it.start();
  const bool any = it.valid();

  auto bar = [&](int i) { return sbase + k64OffBar + 8 * i; };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + k64OffTmemPtr);
  if (threadIdx.x == 0) {
    for (int i = 0; i < k64Stages; ++i) {
      mbar_init(bar(k64BarFull + i), 1);
      mbar_init(bar(k64BarEmpty + i), 1);
    }
    mbar_init(bar(k64BarK), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(k64BarSFull + i), 1);
      mbar_init(bar(k64BarSFree + i), 4);
    }
    mbar_init(bar(k64BarPReady), 4);
    mbar_init(bar(k64BarPFree), 1);
    mbar_init(bar(k64BarAcc), 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.o_map);
    prefetch_tmap(&p.k_map);
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_ptr), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0 && any) {
      const uint64_t pol_k = policy_evict_last(), pol = policy_evict_normal();
      mbar_arrive_expect_tx(bar(k64BarK), k64KBytes);
      tma_load_4d(sbase + k64OffK, &p.k_map, 0, j0, 0, bi, bar(k64BarK), pol_k);
      uint32_t slot = 0, ph = 0;
      auto load_pair = [&](const CUtensorMap* m, int pair, int rb) {
        mbar_wait(bar(k64BarEmpty + slot), ph ^ 1);
        mbar_arrive_expect_tx(bar(k64BarFull + slot), kPairBytes);
        tma_load_4d(sbase + k64OffRing + slot * kPairBytes, m, 0, rb, 2 * pair, bi, bar(k64BarFull + slot), pol);
        if (++slot == k64Stages) {
          slot = 0;
          ph ^= 1;
        }
      };
      // the UMMA issuer's order: the first pass (S, and dP) of tile t + 1 before the gradient pass of tile t
      auto load_first = [&](int rb) {
        if (!kFromP)
          for (int q = 0; q < kQPairs; ++q) load_pair(&p.q_map, q, rb);
        if (!kIsDv)
          for (int q = 0; q < kOPairs; ++q) load_pair(&p.o_map, q, rb);
      };
      auto load_grad = [&](int rb) {
        if (kIsDv)
          for (int q = 0; q < kOPairs; ++q) load_pair(&p.o_map, q, rb);
        else
          for (int q = 0; q < kQPairs; ++q) load_pair(&p.q_map, q, rb);
      };
      RowIter ia = it;
      load_first(ia.rb);
      ia.advance();
      for (; it.valid(); it.advance()) {
        if (ia.valid()) {
          load_first(ia.rb);
          ia.advance();
        }
        load_grad(it.rb);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ UMMA issuer
    if (any) {
      constexpr uint32_t id_s = idesc_bf16_f32(kRows, k64Keys, false, false);
      constexpr uint32_t id_t = idesc_bf16_f32(128, k64Keys, true, true);
      mbar_wait(bar(k64BarK), 0);
      tc_fence_after();
      uint32_t slot = 0, ph = 0;
      auto take = [&]() {
        mbar_wait(bar(k64BarFull + slot), ph);
        tc_fence_after();
      };
      auto release = [&]() {
        if (elect_one()) umma_commit_1sm(bar(k64BarEmpty + slot));
        __syncwarp();
        if (++slot == k64Stages) {
          slot = 0;
          ph ^= 1;
        }
      };
      // S (and dP) of tile t + 1 are issued before the gradient UMMAs of tile t
      auto issue_first = [&](int tc) {
        const int buf = tc % kSBufs, use = tc / kSBufs;
        mbar_wait(bar(k64BarSFree + buf), (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t tS = tmem + kTmemS + 64 * buf;
        for (int q = 0; q < (kFromP ? 0 : kQPairs); ++q) {  // S = Q K^T
          take();
          if (elect_one()) {
            const int nk = q < kQPairs - 1 ? 8 : 4;
            for (int k = 0; k < nk; ++k) {
              const uint32_t ch = 2 * q + (k >> 2), kk = k & 3;
              umma_bf16_1sm(tS, sdesc_sw128(sbase + k64OffRing + slot * kPairBytes + (k >> 2) * 16384 + 32 * kk, 16, 1024),
                            sdesc_sw128(sbase + k64OffK + ch * (k64Keys * 128) + 32 * kk, 16, 1024), id_s, (q | k) != 0);
            }
          }
          release();
        }
        if (!kIsDv) {
          for (int q = 0; q < kOPairs; ++q) {  // dP = dO V^T (V = K[:, :512])
            take();
            if (elect_one()) {
              for (int k = 0; k < 8; ++k) {
                const uint32_t ch = 2 * q + (k >> 2), kk = k & 3;
                umma_bf16_1sm(tmem + kTmemDP + kDPStride * buf,
                              sdesc_sw128(sbase + k64OffRing + slot * kPairBytes + (k >> 2) * 16384 + 32 * kk, 16, 1024),
                              sdesc_sw128(sbase + k64OffK + ch * (k64Keys * 128) + 32 * kk, 16, 1024), id_s,
                              (q | k) != 0);
              }
            }
            release();
          }
        }
        if (elect_one()) umma_commit_1sm(bar(k64BarSFull + buf));
        __syncwarp();
      };
      auto issue_grad = [&](int tc) {
        mbar_wait(bar(k64BarPReady), tc & 1);
        tc_fence_after();
        const uint32_t pb = sbase + k64OffP;
        const int np = kIsDv ? kOPairs : kQPairs;  // dV^T[dims 128 q ..] += dO^T P  /  dK^T[..] += Q^T dS
        for (int q = 0; q < np; ++q) {
          take();
          if (elect_one()) {
            for (int kr = 0; kr < 8; ++kr)
              umma_bf16_1sm(tmem + kTmemAcc + 64 * q,
                            sdesc_sw128(sbase + k64OffRing + slot * kPairBytes + 2048 * kr, 16384, 1024),
                            sdesc_sw128(pb + 2048 * kr, 16, 1024), id_t, (tc | kr) != 0);
          }
          release();
        }
        if (elect_one()) umma_commit_1sm(bar(k64BarPFree));
        __syncwarp();
      };
      RowIter ia = it;
      issue_first(0);
      ia.advance();
      int ta = 1;
      for (int tc = 0; it.valid(); it.advance(), ++tc) {
        if (ia.valid()) {
          issue_first(ta++);
          ia.advance();
        }
        issue_grad(tc);
      }
      if (elect_one()) umma_commit_1sm(bar(k64BarAcc));
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------------ P or dS (thread = row = TMEM lane)
    const int q = warp - 4, row = 32 * q + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const int rows = p.n_q * H;
    const bool jsink = !p.sparse || kb < p.s;
    for (int tc = 0; it.valid(); it.advance(), ++tc) {
      const int buf = tc % kSBufs, use = tc / kSBufs;
      const int r = it.rb + row;
      const bool rv = r < it.re;
      const int rr = rv ? r : 0, t = div_h(p, rr), h = rr - t * H, pos = p.q_start + t;
      const float lse2 = rv ? p.lse[((int64_t)bi * H + h) * p.n_q + t] * kLog2e : 0.f;
      const float Dr = (!kIsDv && rv) ? p.D[(int64_t)bi * rows + rr] : 0.f;
      const bool win = jsink || kb >= pos / p.b - p.l + 1;
      // this row's slots of block kb in the dS row buffer (P from the dV kernel, then dS)
      uint4* dsrow = nullptr;
      if (p.ds && rv) {
        int lbq = pos / p.b - p.l + 1;
        if (lbq < p.s) lbq = p.s;
        const int W = (p.s + p.l) * p.b;
        const int slot = kb < p.s ? j0 : p.s * p.b + (kb - lbq) * p.b + (j0 - kb * p.b);
        dsrow = reinterpret_cast<uint4*>(p.ds + ((int64_t)bi * rows + rr) * W + slot);
      }
      uint32_t pin[32];  // kFromP: P (bf16 pairs), loaded before the dP wait
      if (kFromP) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 x = dsrow ? dsrow[u] : make_uint4(0, 0, 0, 0);
          pin[4 * u] = x.x;
          pin[4 * u + 1] = x.y;
          pin[4 * u + 2] = x.z;
          pin[4 * u + 3] = x.w;
        }
      }
      mbar_wait(bar(k64BarSFull + buf), use & 1);
      tc_fence_after();
      uint32_t pk[32];
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {  // keys 32 hf .. 32 hf + 31
        uint32_t sv[32], dv[32];
        if (!kFromP) tmem_ld32(tl + kTmemS + 64 * buf + 32 * hf, sv);
        if (!kIsDv) tmem_ld32(tl + kTmemDP + kDPStride * buf + 32 * hf, dv);
        tmem_wait_ld();
        if (hf == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_local(bar(k64BarSFree + buf));
        }
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float v2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = j0 + 32 * hf + c + e;
            const bool ok = rv && win && j < p.n_kv && (!p.causal || j <= pos);
            float pv;
            if (kFromP) {
              const uint32_t w2 = pin[16 * hf + (c >> 1)];
              pv = e ? __uint_as_float(w2 & 0xFFFF0000u) : __uint_as_float(w2 << 16);
            } else {
              pv = ok ? ex2(fmaf(__uint_as_float(sv[c + e]), p.sl2, -lse2)) : 0.f;
            }
            v2[e] = kIsDv ? pv : pv * (__uint_as_float(dv[c + e]) - Dr);
          }
          pk[16 * hf + (c >> 1)] = pack_bf16x2(v2[0], v2[1]);
        }
      }
      if (dsrow) {  // this row's 64 values at its slots of block kb: P (dV kernel), dS (dK kernels)
#pragma unroll
        for (int u = 0; u < 8; ++u) dsrow[u] = make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      }
      mbar_wait(bar(k64BarPFree), (tc & 1) ^ 1);
      // row of 128 B = 8 x 16-B units, SWIZZLE_128B: unit u at (u ^ row & 7)
      const uint32_t pr = sbase + k64OffP + row * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        st_shared_v4(pr + (uint32_t)((u ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(k64BarPReady));
    }
    // ------------------------------------------------------------------ epilogue: TMEM lane = dim, column = key
    if (any) {
      mbar_wait(bar(k64BarAcc), 0);
      tc_fence_after();
    }
    const int nm = kIsDv ? kOPairs : kQPairs;
    for (int m = 0; m < nm; ++m) {
      const int dim = 128 * m + 32 * q + lane;
      if (!kIsDv && 128 * m + 32 * q >= kDqk) continue;  // warp-uniform: dims 576.. of the last dK^T tile
      const float sc = kIsDv ? 1.f : p.scale;
#pragma unroll 1
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t v[32];
        if (any) {
          tmem_ld32(tl + kTmemAcc + 64 * m + 32 * hf, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = 0u;
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int j = j0 + 32 * hf + c;
          if (j >= p.n_kv) continue;
          const float x = __uint_as_float(v[c]) * sc;
          if (split) {  // partials in the 32-key tile layout of the sink reduce: [B][n_sink][nsplit][32][1088]
            const int t32 = j >> 5, kl = j & 31;
            p.part[((((int64_t)bi * p.n_sink + t32) * p.nsplit + ys) * kKeys + kl) * kDkv + (kIsDv ? kDqk : 0) + dim] = x;
          } else if (kIsDv) {
            p.dv[((int64_t)bi * p.n_kv + j) * kDv + dim] = x;
          } else {
            p.dk[((int64_t)bi * p.n_kv + j) * kDqk + dim] = x;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

// ------------------------------------------------------------------------ key side, 128-key pair tiles
// The 64-key kernels above move every 128-row tile of Q and dO through one SM per 64 keys (288 KB per tile
// for the dV kernel) and run M128 N64 UMMAs (48 cycles, smem-operand bound). Here a CTA pair (cta_group::2)
// owns the 128 keys of one b-block (b = 128): CTA r stages 64 of them (the N half of every B operand) and
// half of each 128-row tile's operands:
//   dV pair kernel (MODE kPairDv):
//     S   [128 rows x 128 keys] = Q K^T    M128 N128 (A = CTA r's 64 rows of Q, B = its 64 keys); CTA r's TMEM
//                                           holds S of its rows folded: lanes 0-63 keys 0-63, lanes 64-127 keys
//                                           64-127 (64 columns per S buffer, four buffers: S runs three row
//                                           tiles ahead of the gradient UMMAs)
//     P   = exp2(S scale log2e - LSE log2e) by 8 warps per CTA (thread = row x 32 keys); the P of CTA c's keys
//           must end up in CTA c (the N half of the next B operand): the own half is written in place, the
//           other half staged and moved by one 8 KB bulk DSMEM copy. The row's values also go to the dS row
//           buffer (the dK kernel reads P there).
//     dV^T [512 x 128] += dO^T P           M256 N128 per 256-dim group (A = dO^T MN-major: CTA r stages dims
//                                           256 g + 128 r .. + 127 of all 128 rows)
//   dK pair kernel (MODE kPairDk, SSA):
//     dP  = dO V^T                          M128 N128 (A = CTA r's 64 rows of dO, B = V of its 64 keys), two
//                                           buffers
//     dS  = P (dP - D) (P read back from the dS row buffer), into the dS row buffer and, split by keys as above,
//           into the two CTAs' dS buffers
//     dK^T [576 x 128] += Q^T dS            three M256 N128 groups (dims 512.. of the third: CTA 0 stages
//                                           chunk 8 only, CTA 1 nothing; the stale rows are never stored)
// Per SM and 128 x 128 (row, key) pairs the dV kernel moves 136 KB of Q / dO (the 64-key kernel: 576 KB) and
// the dK kernel 144 KB (64-key: 588 KB). TMEM per CTA: dV kernel S 4 x 64 + dV^T 2 x 128 columns; dK kernel
// dK^T 3 x 128 + dP 2 x 64. SMEM: ring 3 x 32 KB, K tile 72 KB (dV: 9 chunks) or 64 KB (dK: V's 8), P / dS
// 2 x 16 KB, staging 2 x 8 KB. Warps 0-7 P / dS and the epilogue (warp w: TMEM lane quarter w % 4, column half w / 4),
// warp 8 TMA, warp 9 UMMA issue (leader) and TMEM allocation, warp 10 the DSMEM copy.
#ifndef PAIR_DS_TMA
#define PAIR_DS_TMA 1
#endif
#ifndef BWD_DK_G2_M128
#define BWD_DK_G2_M128 1
#endif
constexpr int kPairDv = 1, kPairDk = 2;
constexpr int kPKeys = 128, kPHalf = 64;  // keys per pair tile; rows of a 128-row tile per CTA
constexpr int kPThreads = 352, kPProd = 8, kPMma = 9, kPXfer = 10;
template <int MODE>
struct PairCfg {
  static constexpr bool kDv = MODE == kPairDv;
  static constexpr int kStages = 3;
  static constexpr int kKChunks = kDv ? 9 : 8;             // the K tile (S needs 576 dims, dP only V's 512)
  static constexpr int kKBytes = kKChunks * 64 * 128;      // [chunks][64 keys][64 dims]
  static constexpr int kPBytes = kRows * 128;              // P / dS: [128 rows][64 keys] bf16, SW128
  static constexpr int kStBytes = kPHalf * 128;            // staging: [64 rows][the partner's 64 keys]
  // P / dS and staging double-buffered (row tile tc uses buffer tc & 1): the gradient UMMAs of tile tc - 1
  // and the DSMEM copy of tile tc overlap the P of tile tc + 1
  static constexpr int kOffRing = 0, kOffK = kStages * kPairBytes, kOffP = kOffK + kKBytes,
                       kOffSt = kOffP + 2 * kPBytes, kOffBar = kOffSt + 2 * kStBytes;
  // S / dP buffers and the first-pass lookahead (dK: dK^T's third dim group as an M128 UMMA takes 64 columns,
  // which leaves room for a third dP buffer)
  static constexpr int kSBufs = kDv ? 4 : (BWD_DK_G2_M128 ? 3 : 2), kAhead = kSBufs - 1;
  static constexpr int kBarFull = 0, kBarEmpty = kStages, kBarK = 2 * kStages, kBarSFull = kBarK + 1,
                       kBarSFree = kBarSFull + kSBufs, kBarPLocal = kBarSFree + kSBufs, kBarPStaged = kBarPLocal + 2,
                       kBarPRecv = kBarPStaged + 2, kBarPFull = kBarPRecv + 2, kBarPFree = kBarPFull + 2,
                       kBarPStored = kBarPFree + 2, kBarAcc = kBarPStored + 2, kNumBars = kBarAcc + 1;
  static constexpr int kOffTmemPtr = kOffBar + 8 * kNumBars;
  static constexpr int kSmem = kOffTmemPtr + 16 + 1024;
  static constexpr int kFirstItems = kDv ? 3 : 2;  // Q (chunks 0-3, 4-7, 8) or dO (0-3, 4-7) of this CTA's 64 rows
  static constexpr int kGroups = kDv ? 2 : 3;      // 256-dim M groups of dV^T / dK^T
  static constexpr uint32_t kTmemS = kDv ? 0 : (BWD_DK_G2_M128 ? 320 : 384), kTmemAcc = kDv ? 256 : 0;
};
static_assert(PairCfg<kPairDv>::kSmem <= 232448 && PairCfg<kPairDk>::kSmem <= 232448, "smem");

// clock64 timeline: trace[(slot * 2 + rank) * 64 + tile] for tiles < 64 of pair cluster trace_cluster
#define BTRACE(slot, idx)                                                                                   \
  do {                                                                                                      \
    if (p.trace && pc == p.trace_cluster && (idx) < 64 && (threadIdx.x & 31) == 0)                          \
      p.trace[((slot) * 2 + rank) * 64 + (idx)] = clock64();                                                \
  } while (0)

template <int MODE>
__global__ void __launch_bounds__(kPThreads, 1) __cluster_dims__(2, 1, 1)
    bwd_pair_tc_kernel(const __grid_constant__ TcBwdParams p) {
  using C = PairCfg<MODE>;
  constexpr bool kDvK = C::kDv;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sbase - sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank(), partner = rank ^ 1u;
  const int H = p.heads;
  const int ktiles = (p.n_kv + kPKeys - 1) / kPKeys;
  // clusters of a batch entry: the sink tiles' row splits first (they are as long as a full local tile and must
  // not start late), then the local tiles, each in p.lsplit row splits (short sequences: fill the SMs)
  const int ns = p.sparse ? (p.s < ktiles ? p.s : ktiles) : 0;  // sink tiles (nsplit units each, 1 if unsplit)
  const int units = ns * p.nsplit + (ktiles - ns) * p.lsplit;
  const int pc = (int)(blockIdx.x >> 1);
  const int bi = pc / units, u = pc - bi * units;
  const bool sink_unit = u < ns * p.nsplit;
  const int tile = sink_unit ? u / p.nsplit : ns + (u - ns * p.nsplit) / p.lsplit;
  const int ys = sink_unit ? u - tile * p.nsplit : (u - ns * p.nsplit) % p.lsplit;  // row split of the tile
  const int j0 = tile * kPKeys;
  // rows attending keys [j0, j0 + 128) (b == 128: the tile is one block)
  int p0 = p.causal ? j0 : 0, p1 = p.q_start + p.n_q;
  const int kb = j0 / p.b;
  if (p.sparse && kb >= p.s) {
    const int pe = (kb + p.l) * p.b;
    if (pe < p1) p1 = pe;
  }
  if (p0 < p.q_start) p0 = p.q_start;
  const bool split = p.sparse && kb < p.s && p.nsplit > 1;
  const bool lsplit = p.sparse && kb >= p.s && p.lsplit > 1;  // a local tile's row split: partials too
  if (split || lsplit) {  // rows split by whole query blocks, walked in the local tiles' rotation
    if (p1 > p0) {
      const int nsp = split ? p.nsplit : p.lsplit;
      const int ma = p0 / p.b, nb = (p1 - 1) / p.b - ma + 1, cb = (nb + nsp - 1) / nsp;
      const int a = (ma + ys * cb) * p.b, e = a + cb * p.b;
      if (a > p0) p0 = a;
      if (e < p1) p1 = e;
    }
  }
  RowIter it;
  it.L = p.sparse && (split || kb >= p.s) ? p.l : 1;
  it.m0 = p0 / p.b;
  it.m1 = (p1 - 1) / p.b;
  it.p0 = p0;
  it.p1 = p1;
  it.R0 = p1 > p0 ? (p0 - p.q_start) * H : 0;
  it.R1 = p1 > p0 ? (p1 - p.q_start) * H : 0;
  it.qs = p.q_start;
  it.H = H;
  it.b = p.b;
  it.start();
  const bool any = it.valid();
  // debug (trace_cluster < 0): globaltimer at start / end of every cluster, [pc][2] (rank 0, thread 0)
  const bool gtrace = p.trace && p.trace_cluster < 0 && rank == 0 && threadIdx.x == 0;
  if (gtrace) {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    p.trace[(int64_t)pc * 2] = g;
  }
  // the tile's P / dS rows go to the dS row buffer by one TMA store of this CTA's key half (the operand buffer
  // is already [128 rows][64 keys] swizzled, the box's layout) when all 128 rows are the segment's or the
  // tensor ends inside the tile (the store clips there); otherwise by per-thread stores
  const int rows_total = p.n_q * H;
  auto tma_rows = [&](const RowIter& ri) {
    return PAIR_DS_TMA && p.ds != nullptr && (ri.rb + kRows <= ri.re || ri.re == rows_total);
  };

  auto bar = [&](int i) { return sbase + C::kOffBar + 8 * i; };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::kOffTmemPtr);
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(bar(C::kBarFull + i), 1);
      mbar_init(bar(C::kBarEmpty + i), 1);
    }
    mbar_init(bar(C::kBarK), 1);
    for (int i = 0; i < C::kSBufs; ++i) {
      mbar_init(bar(C::kBarSFull + i), 1);
      mbar_init(bar(C::kBarSFree + i), 16);  // 8 warps of each CTA (leader's barrier)
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(C::kBarPLocal + i), 4);
      mbar_init(bar(C::kBarPStaged + i), 4);
      mbar_init(bar(C::kBarPRecv + i), 1);
      mbar_init(bar(C::kBarPFull + i), 2);  // the transfer warp of each CTA (leader's barrier)
      mbar_init(bar(C::kBarPFree + i), 1);
      mbar_init(bar(C::kBarPStored + i), 1);  // the transfer warp: the TMA store of the tile's rows read P
    }
    mbar_init(bar(C::kBarAcc), 1);
    fence_mbar_init();
    RowIter i1 = it;  // tiles 0 and 1: the partner's rows, armed ahead
    for (int i = 0; i < 2 && i1.valid(); ++i, i1.advance()) mbar_arrive_expect_tx(bar(C::kBarPRecv + i), C::kStBytes);
  }
  if (warp == kPProd && lane == 0) {
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.o_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(kDvK ? &p.q4_map : &p.o4_map);
    prefetch_tmap(&p.q1_map);
  }
  if (warp == kPMma) tmem_alloc<2>(smem_u32(tmem_ptr), 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;

  if (warp == kPProd) {
    // ------------------------------------------------------------------ TMA producer (each CTA)
    if (any) {
      const uint64_t pol_k = policy_evict_last(), pol = policy_evict_normal();
      const uint32_t full_l = mapa(bar(C::kBarFull), 0);
      if (elect_one()) {
        if (rank == 0) mbar_arrive_expect_tx(bar(C::kBarK), 2 * C::kKBytes);
        tma_load_4d_pair(sbase + C::kOffK, &p.k_map, 0, j0 + 64 * (int)rank, 0, bi, mapa(bar(C::kBarK), 0), pol_k);
      }
      __syncwarp();
      uint32_t slot = 0, ph = 0;
      // tx: the bytes both CTAs load into this slot; mine: whether this CTA loads (m, row, chunk)
      auto load = [&](const CUtensorMap* m, int row, int chunk, uint32_t tx, bool mine = true) {
        mbar_wait(bar(C::kBarEmpty + slot), ph ^ 1);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(C::kBarFull + slot), tx);
          if (mine) tma_load_4d_pair(sbase + C::kOffRing + slot * kPairBytes, m, 0, row, chunk, bi, full_l + 8 * slot, pol);
        }
        __syncwarp();
        if (++slot == C::kStages) {
          slot = 0;
          ph ^= 1;
        }
      };
      // first pass: this CTA's 64 rows ([4 chunks][64 rows] boxes: Q for S, or dO for dP); gradient pass: the
      // tile's 128 rows of this CTA's dims of each 256-dim group ([2 chunks][128 rows]: dO for dV^T, Q for dK^T)
      auto load_first = [&](int rb) {
        const int r = rb + kPHalf * (int)rank;
        if (kDvK) {
          load(&p.q4_map, r, 0, 2 * kPairBytes);
          load(&p.q4_map, r, 4, 2 * kPairBytes);
          load(&p.q1_map, r, 8, 2 * kPairBytes / 4);
        } else {
          load(&p.o4_map, r, 0, 2 * kPairBytes);
          load(&p.o4_map, r, 4, 2 * kPairBytes);
        }
      };
      auto load_grad = [&](int rb) {
        for (int g = 0; g < 2; ++g) load(kDvK ? &p.o_map : &p.q_map, rb, 2 * (2 * g + (int)rank), 2 * kPairBytes);
        // dK^T's third group, dims 512..: CTA 0 stages chunk 8 alone ([1 chunk][128 rows], p.q1_map of the dK
        // kernel), CTA 1 nothing; the UMMA rows they leave stale (dims 576..) are never stored
        if (!kDvK) load(&p.q1_map, rb, 8, kPairBytes / 2, rank == 0);
      };
      RowIter ia = it;
      for (int i = 0; i < C::kAhead && ia.valid(); ++i) {
        load_first(ia.rb);
        ia.advance();
      }
      for (RowIter ib = it; ib.valid(); ib.advance()) {
        if (ia.valid()) {
          load_first(ia.rb);
          ia.advance();
        }
        load_grad(ib.rb);
      }
      // drain: the last commits to this CTA's Empty barriers land before it can exit
      for (int i = 0; i < C::kStages; ++i) {
        mbar_wait(bar(C::kBarEmpty + slot), ph ^ 1);
        if (++slot == C::kStages) {
          slot = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == kPMma) {
    // ------------------------------------------------------------------ UMMA issuer (leader CTA)
    if (any && rank == 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(128, kPKeys, false, false);
      constexpr uint32_t id_t = idesc_bf16_f32(256, kPKeys, true, true);
      mbar_wait(bar(C::kBarK), 0);
      tc_fence_after();
      uint32_t slot = 0, ph = 0;
      auto take = [&]() {
        mbar_wait(bar(C::kBarFull + slot), ph);
        tc_fence_after();
      };
      auto release = [&]() {
        if (elect_one()) umma_commit_pair_mc(bar(C::kBarEmpty + slot), 3);
        __syncwarp();
        if (++slot == C::kStages) {
          slot = 0;
          ph ^= 1;
        }
      };
      // S = Q K^T (dV kernel) or dP = dO V^T (dK kernel) of row tile tc into buffer tc % kSBufs
      auto issue_first = [&](int tc) {
        const int buf = tc % C::kSBufs, use = tc / C::kSBufs;
        BTRACE(0, tc);
        mbar_wait(bar(C::kBarSFree + buf), (use & 1) ^ 1);
        BTRACE(1, tc);
        tc_fence_after();
        const uint32_t d = tmem + C::kTmemS + 64 * buf;
        for (int q = 0; q < C::kFirstItems; ++q) {
          take();
          if (elect_one()) {
            const int nk = q < 2 ? 16 : 4;  // 4 chunks x 4 k steps (the dV kernel's third item: chunk 8 alone)
            for (int k = 0; k < nk; ++k) {
              const uint32_t ch = 4 * q + (k >> 2), kk = k & 3;
              umma_bf16_pair(d, sdesc_sw128(sbase + C::kOffRing + slot * kPairBytes + (k >> 2) * (kPHalf * 128) + 32 * kk, 16, 1024),
                             sdesc_sw128(sbase + C::kOffK + ch * (64 * 128) + 32 * kk, 16, 1024), id_s, (q | k) != 0);
            }
          }
          release();
        }
        if (elect_one()) umma_commit_pair_mc(bar(C::kBarSFull + buf), 3);
        __syncwarp();
        BTRACE(2, tc);
      };
      // dV^T += dO^T P or dK^T += Q^T dS over the tile's 128 rows (P / dS rows 64 c .. from CTA c)
      auto issue_grad = [&](int tc) {
        BTRACE(3, tc);
        mbar_wait_acquire_cluster(bar(C::kBarPFull + (tc & 1)), (tc >> 1) & 1);  // both CTAs' P halves are in place
        BTRACE(4, tc);
        tc_fence_after();
        const uint32_t pb = sbase + C::kOffP + (tc & 1) * C::kPBytes;
        for (int g = 0; g < C::kGroups; ++g) {
          // dK^T dims 512..575 (CTA 0's one chunk): an M128 UMMA, 64 rows per CTA, D folded over the lanes
          const bool m128 = !kDvK && BWD_DK_G2_M128 && g == 2;
          constexpr uint32_t id_t2 = idesc_bf16_f32(128, kPKeys, true, true);
          take();
          if (elect_one()) {
            for (int kr = 0; kr < 8; ++kr)
              umma_bf16_pair(tmem + C::kTmemAcc + 128 * g,
                             sdesc_sw128(sbase + C::kOffRing + slot * kPairBytes + 2048 * kr, 16384, 1024),
                             sdesc_sw128(pb + 2048 * kr, 16, 1024), m128 ? id_t2 : id_t, (tc | kr) != 0);
          }
          release();
        }
        if (elect_one()) umma_commit_pair_mc(bar(C::kBarPFree + (tc & 1)), 3);
        __syncwarp();
        BTRACE(5, tc);
      };
      RowIter ia = it;
      int ta = 0, tc = 0;
      for (; ta < C::kAhead && ia.valid(); ++ta, ia.advance()) issue_first(ta);
      for (RowIter ib = it; ib.valid(); ib.advance(), ++tc) {
        if (ia.valid()) {
          issue_first(ta++);
          ia.advance();
        }
        issue_grad(tc);
      }
      if (elect_one()) umma_commit_pair_mc(bar(C::kBarAcc), 3);
      __syncwarp();
      // the last buffer releases (remote arrivals from the partner) land before this CTA can exit
      for (int u = ta - C::kSBufs; u < ta; ++u)
        if (u >= 0) mbar_wait(bar(C::kBarSFree + u % C::kSBufs), (u / C::kSBufs) & 1);
    }
  } else if (warp == kPXfer) {
    // ------------------------------------------------------------------ the staged half to the partner
    if (any) {
      const uint32_t pfull0 = mapa(bar(C::kBarPFull), 0);
      const uint32_t dst = mapa(sbase + C::kOffP + (uint32_t)(kPHalf * rank) * 128, partner);
      const uint32_t precv = mapa(bar(C::kBarPRecv), partner);
      RowIter ix = it;
      for (int tc = 0; ix.valid(); ix.advance(), ++tc) {
        const uint32_t pb = (uint32_t)tc & 1, ph = ((uint32_t)tc >> 1) & 1;
        mbar_wait(bar(C::kBarPStaged + pb), ph);
        if (lane == 0)
          bulk_copy_to_cluster(dst + pb * C::kPBytes, sbase + C::kOffSt + pb * C::kStBytes, C::kStBytes, precv + 8 * pb);
        mbar_wait_spin(bar(C::kBarPRecv + pb), ph);  // the partner's rows of this CTA's half landed
        mbar_wait(bar(C::kBarPLocal + pb), ph);      // and this CTA's own rows are written
        if (lane == 0) {
          RowIter n2 = ix;
          n2.advance();
          n2.advance();
          if (n2.valid()) mbar_arrive_expect_tx(bar(C::kBarPRecv + pb), C::kStBytes);  // tile tc + 2's, armed ahead
          mbar_arrive_release_cluster(pfull0 + 8 * pb);
          if (tma_rows(ix)) {  // this CTA's 64 keys of the tile's 128 rows, from the complete operand buffer
            const int t0 = div_h(p, ix.rb), QB = (p.q_start + t0) / p.b;
            int lbq = QB - p.l + 1;
            if (lbq < p.s) lbq = p.s;
            const int slot = (kb < p.s ? j0 : p.s * p.b + (kb - lbq) * p.b) + 64 * (int)rank;
            tma_store_3d(&p.ds_map, sbase + C::kOffP + pb * C::kPBytes, slot, ix.rb, bi);
            bulk_commit_group();
            bulk_wait_group_read0();
          }
          mbar_arrive_local(bar(C::kBarPStored + pb));  // buffer pb may take tile tc + 2
        }
        __syncwarp();
      }
      if (lane == 0) bulk_wait_group0();
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------------ P or dS (thread = row x 32 keys)
    // TMEM lane quarter q: rows 32 (q & 1) .., key half kh = q >> 1 (the fold of the M128 D); column half c
    const int q = warp & 3, c = warp >> 2, kh = q >> 1, row = 32 * (q & 1) + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    const int rows = p.n_q * H;
    const bool jsink = !p.sparse || kb < p.s;
    const bool own = kh == (int)rank;  // keys 64 kh .. belong to CTA kh
    const int jk = j0 + 64 * kh + 32 * c;  // this thread's first key
    const uint32_t sfree0 = mapa(bar(C::kBarSFree), 0);
    // this row's P in buffer 0 (buffer 1: + kPBytes / kStBytes)
    const uint32_t pdst = own ? sbase + C::kOffP + (uint32_t)(kPHalf * rank + row) * 128 : sbase + C::kOffSt + row * 128;
    const uint32_t pstride = own ? C::kPBytes : C::kStBytes;
    const uint32_t sw = (uint32_t)(row & 7);
    struct RowIn {
      bool rv, win;
      int pos;
      float lse2, Dr;
      uint4* ds;  // this row's 32 slots (keys jk ..) of block kb in the dS row buffer
      bool tma;   // the tile's rows are written by the transfer warp's TMA store
    };
    auto row_in = [&](const RowIter& ri) {
      RowIn x;
      const int r = ri.rb + kPHalf * (int)rank + row;
      x.rv = ri.valid() && r < ri.re;
      const int rr = x.rv ? r : 0, t = div_h(p, rr), h = rr - t * H;
      x.pos = p.q_start + t;
      x.lse2 = (kDvK && x.rv) ? p.lse[((int64_t)bi * H + h) * p.n_q + t] * kLog2e : 0.f;
      x.Dr = (!kDvK && x.rv) ? p.D[(int64_t)bi * rows + rr] : 0.f;
      x.win = jsink || kb >= x.pos / p.b - p.l + 1;
      x.ds = nullptr;
      x.tma = tma_rows(ri);
      if (p.ds && x.rv) {
        int lbq = x.pos / p.b - p.l + 1;
        if (lbq < p.s) lbq = p.s;
        const int W = (p.s + p.l) * p.b;
        const int slot = (kb < p.s ? j0 : p.s * p.b + (kb - lbq) * p.b) + (jk - j0);
        x.ds = reinterpret_cast<uint4*>(p.ds + ((int64_t)bi * rows + rr) * W + slot);
      }
      return x;
    };
    uint32_t pn[16];  // dK kernel: the next tile's P (bf16 pairs), loaded one tile ahead
    auto load_p = [&](const RowIn& x) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 v = x.ds ? x.ds[u] : make_uint4(0, 0, 0, 0);
        pn[4 * u] = v.x;
        pn[4 * u + 1] = v.y;
        pn[4 * u + 2] = v.z;
        pn[4 * u + 3] = v.w;
      }
    };
    RowIn cur = row_in(it);
    if (!kDvK) load_p(cur);
    uint4* prev_ds = nullptr;  // the previous tile's dS row slots, stored one tile late: a proxy fence waits
    uint32_t prev[16];         // for this thread's outstanding global stores
    int tc = 0;
    for (; it.valid(); ++tc) {
      const int buf = tc % C::kSBufs, use = tc / C::kSBufs;
      uint32_t pk[16];
      if (!kDvK) {
#pragma unroll
        for (int u = 0; u < 16; ++u) pk[u] = pn[u];
      }
      RowIter nx = it;
      nx.advance();
      const RowIn nxt = row_in(nx);  // the next tile's row inputs (and P) while this tile is processed
      if (!kDvK) load_p(nxt);
      mbar_wait(bar(C::kBarSFull + buf), use & 1);
      if (warp == 0) BTRACE(6, tc);
      tc_fence_after();
      uint32_t sv[32];
      tmem_ld32(tl + C::kTmemS + 64 * buf + 32 * c, sv);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(sfree0 + 8 * buf);
      if (warp == 0) BTRACE(7, tc);
#pragma unroll
      for (int e2 = 0; e2 < 32; e2 += 2) {
        float v2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = jk + e2 + e;
          const bool ok = cur.rv && cur.win && j < p.n_kv && (!p.causal || j <= cur.pos);
          if (kDvK) {
            v2[e] = ok ? ex2(fmaf(__uint_as_float(sv[e2 + e]), p.sl2, -cur.lse2)) : 0.f;
          } else {
            const uint32_t w2 = pk[e2 >> 1];
            const float pv = e ? __uint_as_float(w2 & 0xFFFF0000u) : __uint_as_float(w2 << 16);
            v2[e] = pv * (__uint_as_float(sv[e2 + e]) - cur.Dr);
          }
        }
        pk[e2 >> 1] = pack_bf16x2(v2[0], v2[1]);
      }
      if (warp == 0) BTRACE(8, tc);
      const int pb = tc & 1;
      mbar_wait(bar(C::kBarPFree + pb), ((tc >> 1) & 1) ^ 1);  // buffer pb's last gradient UMMAs (tile tc - 2) ran
      mbar_wait(bar(C::kBarPStored + pb), ((tc >> 1) & 1) ^ 1);  // and the TMA store of tile tc - 2's rows read it
      if (warp == 0) BTRACE(9, tc);
      // row of 128 B = 8 x 16-B units (this thread's: 4 c .. 4 c + 3), SWIZZLE_128B: unit u at (u ^ row & 7)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        st_shared_v4(pdst + pb * pstride + (((4 * c + u) ^ sw) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2],
                     pk[4 * u + 3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar((own ? C::kBarPLocal : C::kBarPStaged) + pb));
      if (warp == 0) BTRACE(10, tc);
      if (prev_ds) {  // P (dV kernel) or dS (dK kernel) of the previous tile's row, 32 keys, to the dS row buffer
#pragma unroll
        for (int u = 0; u < 4; ++u) prev_ds[u] = make_uint4(prev[4 * u], prev[4 * u + 1], prev[4 * u + 2], prev[4 * u + 3]);
      }
      prev_ds = cur.tma ? nullptr : cur.ds;
#pragma unroll
      for (int u = 0; u < 16; ++u) prev[u] = pk[u];
      it = nx;
      cur = nxt;
    }
    if (prev_ds) {
#pragma unroll
      for (int u = 0; u < 4; ++u) prev_ds[u] = make_uint4(prev[4 * u], prev[4 * u + 1], prev[4 * u + 2], prev[4 * u + 3]);
    }
    // ------------------------------------------------------------------ epilogue: TMEM lane = dim, column = key
    if (any) {
      for (int u = tc - 2 < 0 ? 0 : tc - 2; u < tc; ++u)  // the last gradient commits (they precede Acc) landed
        mbar_wait(bar(C::kBarPFree + (u & 1)), (u >> 1) & 1);
      mbar_wait(bar(C::kBarAcc), 0);
      tc_fence_after();
    }
    for (int g = 0; g < C::kGroups; ++g) {
      const bool m128 = !kDvK && BWD_DK_G2_M128 && g == 2;
      // M256 groups: lane = dim 256 g + 128 rank + lane, column = key. The M128 group (dims 512..575, CTA 0):
      // lanes 0-63 hold the dims for keys 0-63, lanes 64-127 the same dims for keys 64-127
      const int d0 = m128 ? (rank == 0 ? 512 + 32 * (q & 1) : kDqk) : 256 * g + 128 * (int)rank + 32 * q;
      const int dim = d0 + lane;
      if (d0 >= (kDvK ? kDv : kDqk)) continue;  // warp-uniform: the zero-filled dims of dK^T's third group
      const float sc = kDvK ? 1.f : p.scale;
#pragma unroll 1
      for (int hf = 0; hf < (m128 ? 1 : 2); ++hf) {
        uint32_t v[32];
        if (any) {
          tmem_ld32(tl + C::kTmemAcc + 128 * g + (m128 ? 32 * c : 64 * c + 32 * hf), v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = 0u;
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int j = j0 + (m128 ? 64 * (q >> 1) + 32 * c : 64 * c + 32 * hf) + e;
          if (j >= p.n_kv) continue;
          const float x = __uint_as_float(v[e]) * sc;
          if (split) {  // partials in the 32-key tile layout of the sink reduce: [B][n_sink][nsplit][32][1088]
            const int t32 = j >> 5, kl = j & 31;
            p.part[((((int64_t)bi * p.n_sink + t32) * p.nsplit + ys) * kKeys + kl) * kDkv + (kDvK ? kDqk : 0) + dim] = x;
          } else if (lsplit) {  // [B][kt - ns][lsplit][128][1088]
            p.part_local[((((int64_t)bi * (ktiles - ns) + (tile - ns)) * p.lsplit + ys) * kPKeys + (j - j0)) * kDkv +
                         (kDvK ? kDqk : 0) + dim] = x;
          } else if (kDvK) {
            p.dv[((int64_t)bi * p.n_kv + j) * kDv + dim] = x;
          } else {
            p.dk[((int64_t)bi * p.n_kv + j) * kDqk + dim] = x;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (gtrace) {
    uint64_t g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    p.trace[(int64_t)pc * 2 + 1] = g;
  }
  if (warp == kPMma) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}

// dK, dV of the local tiles that ran in row splits: the fixed-order sum of their partials
__global__ void __launch_bounds__(256) bwd_local_reduce_kernel(const float* __restrict__ part, float* dk, float* dv,
                                                               int32_t batch, int32_t n_kv, int32_t ns, int32_t nloc,
                                                               int32_t lsplit) {
  const int64_t per = (int64_t)nloc * kPKeys * (kDkv / 4);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)batch * per) return;
  const int bi = (int)(i / per);
  const int64_t rem = i - bi * per;
  const int t = (int)(rem / (kPKeys * (kDkv / 4)));
  const int r2 = (int)(rem - (int64_t)t * kPKeys * (kDkv / 4));
  const int kl = r2 / (kDkv / 4), c = 4 * (r2 - kl * (kDkv / 4));
  const int j = (ns + t) * kPKeys + kl;
  if (j >= n_kv) return;
  const float* src = part + ((((int64_t)bi * nloc + t) * lsplit) * kPKeys + kl) * kDkv + c;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int y = 0; y < lsplit; ++y) {
    const float4 v = *reinterpret_cast<const float4*>(src + (int64_t)y * kPKeys * kDkv);
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  float* dst = c < kDqk ? dk + ((int64_t)bi * n_kv + j) * kDqk + c : dv + ((int64_t)bi * n_kv + j) * kDv + c - kDqk;
  *reinterpret_cast<float4*>(dst) = s;
}

// ---------------------------------------------------------------------------------------------- dQ = dS K
// SSA only: dQ[128 rows, 192-dim slice] = scale * DS[rows, slots] K[slots -> keys, slice] as a tcgen05 GEMM
// (M128 N192 K16, A = DS K-major, B = K MN-major over 3 64-dim atoms) from the dS rows the key kernel wrote:
// the rows of a tile share one query block (tokens of one b-block), hence one slot -> key map: slots [0, s b)
// are the sink keys, slots s b + i the keys lbq b + i of the local window (lbq = max(s, QB - l + 1)).
constexpr int kQdN = 192, kQdStages = 4;
constexpr int kQdA = kRows * 128;          // [128 rows][64 slots] bf16, SW128
constexpr int kQdB = 3 * 64 * 128;         // [3 chunks][64 keys][64 dims], SW128
constexpr int kQdStage = kQdA + kQdB;      // 40 KB
constexpr int kQdOffSt = kQdStages * kQdStage;       // epilogue staging: 4 warps x 2 x [32 rows][32 fp32], SW128
constexpr int kQdStBytes = 32 * 128;
constexpr int kQdOffBar = kQdOffSt + 4 * 2 * kQdStBytes;
constexpr int kQdNumBars = 2 * kQdStages + 4;
constexpr int kQdOffTmemPtr = kQdOffBar + 8 * kQdNumBars;
constexpr int kQdSmem = kQdOffTmemPtr + 16 + 1024;

struct TcDqParams {
  CUtensorMap ds_map;  // 3-D {W slots, rows, B}, box {64, 128, 1}
  CUtensorMap k_map;   // 4-D {64, n_kv, 9, B}, box {64, 64, 3, 1}
  CUtensorMap dq_map;  // 3-D fp32 {576, rows, B}, box {32, 32, 1}, SW128 (epilogue TMA stores)
  float* dq;
  int32_t rows, heads, n_kv, q_start, s, l, b, kv32, batch;
  float scale;
  uint32_t h_m, h_p;
};

__global__ void __launch_bounds__(256, 1) bwd_dq_tc_kernel(const __grid_constant__ TcDqParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sbase - sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rtiles = (p.rows + kRows - 1) / kRows;
  const int ntiles = p.batch * rtiles * 3;
  // Persistent: tiles (128 rows, 192-dim slice) strided over the grid; the dQ accumulator is double-buffered
  // in TMEM (2 x 192 columns) so a tile's epilogue overlaps the next tile's loads and MMAs.
  struct Tile {
    int bi, r0, slice, lbq, se, nl, nsc, nch;
  };
  auto decode = [&](int t) {
    Tile T;
    T.slice = t % 3;
    const int rest = t / 3;
    T.bi = rest / rtiles;
    T.r0 = (rest - T.bi * rtiles) * kRows;
    const int t0 = (int)(((uint64_t)(uint32_t)T.r0 * p.h_m) >> p.h_p), QB = (p.q_start + t0) / p.b;
    T.lbq = QB - p.l + 1 < p.s ? p.s : QB - p.l + 1;
    // Slots the key kernel wrote for every row of the tile: keys below the 32-key boundary after the tile's
    // last position (a tile's 128 / H <= 32 tokens never straddle such a boundary; keys past a row's own
    // position inside it carry dS = 0). Beyond it a row was never visited by the key tile's CTA.
    const int rl = T.r0 + kRows - 1 < p.rows ? T.r0 + kRows - 1 : p.rows - 1;
    const int tl = (int)(((uint64_t)(uint32_t)rl * p.h_m) >> p.h_p);
    const int lim = (p.q_start + tl + 1 + 31) / 32 * 32;
    T.se = p.s * p.b < lim ? p.s * p.b : lim;
    const int hil = (QB + 1) * p.b < lim ? (QB + 1) * p.b : lim;
    T.nl = hil > T.lbq * p.b ? hil - T.lbq * p.b : 0;
    T.nsc = (T.se + 63) / 64;
    T.nch = T.nsc + (T.nl + 63) / 64;
    return T;
  };
  // chunk c of a tile: first slot, first key, k steps (16 slots each)
  auto chunk = [&](const Tile& T, int c, int& slot, int& key, int& nk) {
    if (c < T.nsc) {
      slot = key = 64 * c;
      nk = (T.se - 64 * c) >= 64 ? 4 : (T.se - 64 * c) / 16;
    } else {
      const int i = 64 * (c - T.nsc);
      slot = p.s * p.b + i;
      key = T.lbq * p.b + i;
      nk = (T.nl - i) >= 64 ? 4 : (T.nl - i) / 16;
    }
  };
  // barriers: Full[kQdStages], Empty[kQdStages], AccFull[2], AccFree[2]
  auto bar = [&](int i) { return sbase + kQdOffBar + 8 * i; };
  const int kAccFull = 2 * kQdStages, kAccFree = kAccFull + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + kQdOffTmemPtr);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kQdStages; ++i) {
      mbar_init(bar(i), 1);
      mbar_init(bar(kQdStages + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kAccFull + i), 1);
      mbar_init(bar(kAccFree + i), 4);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.ds_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(&p.dq_map);
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_ptr), 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_normal(), pol_k = policy_evict_last();
      uint32_t slot = 0, ph = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = decode(t);
        for (int c = 0; c < T.nch; ++c) {
          int sl, key, nk;
          chunk(T, c, sl, key, nk);
          mbar_wait(bar(kQdStages + slot), ph ^ 1);
          mbar_arrive_expect_tx(bar(slot), kQdStage);
          const uint32_t dst = sbase + slot * kQdStage;
          tma_load_3d(dst, &p.ds_map, sl, T.r0, T.bi, bar(slot), pol);
          tma_load_4d(dst + kQdA, &p.k_map, 0, key, 3 * T.slice, T.bi, bar(slot), pol_k);
          if (++slot == kQdStages) {
            slot = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id = idesc_bf16_f32(kRows, kQdN, false, true);
    uint32_t slot = 0, ph = 0;
    int n = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
      const Tile T = decode(t);
      const int ab = n & 1, use = n >> 1;
      mbar_wait(bar(kAccFree + ab), (use & 1) ^ 1);
      tc_fence_after();
      for (int c = 0; c < T.nch; ++c) {
        int sl, key, nk;
        chunk(T, c, sl, key, nk);
        mbar_wait(bar(slot), ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a = sbase + slot * kQdStage;
          for (int k = 0; k < nk; ++k)
            umma_bf16_1sm(tmem + kQdN * ab, sdesc_sw128(a + 32 * k, 16, 1024), sdesc_sw128(a + kQdA + 2048 * k, 8192, 1024),
                          id, (c | k) != 0);
          umma_commit_1sm(bar(kQdStages + slot));
        }
        __syncwarp();
        if (++slot == kQdStages) {
          slot = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit_1sm(bar(kAccFull + ab));
      __syncwarp();
    }
  } else if (warp >= 4) {
    // a row's 32 values per TMEM load into a swizzled [32 rows][32 fp32] staging block, then one TMA store of
    // 32 full 128-B row pieces (per-thread row stores wrote half sectors and queued behind each other)
    const int q = warp - 4, row = 32 * q + lane;
    const uint32_t st0 = sbase + kQdOffSt + (uint32_t)q * 2 * kQdStBytes, sw = (uint32_t)(lane & 7);
    int n = 0, k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++n) {
      const Tile T = decode(t);
      const int ab = n & 1, use = n >> 1;
      mbar_wait(bar(kAccFull + ab), use & 1);
      tc_fence_after();
      for (int g = 0; g < kQdN / 32; ++g, ++k) {
        uint32_t v[32];
        if (T.nch > 0) {
          tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + kQdN * ab + 32 * g, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = 0u;
        }
        if (g == kQdN / 32 - 1) {  // the accumulator is read: the next-but-one tile may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_local(bar(kAccFree + ab));
        }
        const uint32_t sb = st0 + (uint32_t)(k & 1) * kQdStBytes;
        if (lane == 0) bulk_wait_group_read1();  // the store that last read this staging block is done
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 8; ++u)
          st_shared_v4(sb + lane * 128 + ((u ^ sw) << 4), __float_as_uint(__uint_as_float(v[4 * u]) * p.scale),
                       __float_as_uint(__uint_as_float(v[4 * u + 1]) * p.scale),
                       __float_as_uint(__uint_as_float(v[4 * u + 2]) * p.scale),
                       __float_as_uint(__uint_as_float(v[4 * u + 3]) * p.scale));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {  // rows past p.rows are clipped by the tensor map
          tma_store_3d(&p.dq_map, sb, kQdN * T.slice + 32 * g, T.r0 + 32 * q, T.bi);
          bulk_commit_group();
        }
      }
      (void)row;
    }
    if (lane == 0) bulk_wait_group0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

// dQ = dS K on CTA pairs (cta_group::2), when the key side ran the 128-key pair kernels (every slot of the blocks
// up to a row's own was written for every row of its block) and 256-row tiles stay in one query block:
// a pair tile = 256 rows (CTA r: 128, the M half) x a 256-dim slice (CTA r stages 128 of the slice's dims, the
// N half of B): M256 N256 K16 UMMAs (the third slice, dims 512..575, N128 with CTA 1's half out of range). Per
// CTA and 64 slots: 16 KB of dS + 16 KB of K for 512 tensor cycles (the single-CTA M128 N192 kernel: 40 KB per
// 384). Six 32 KB stages; the epilogue's TMA stores as in bwd_dq_tc_kernel.
constexpr int kQpStages = 6;
constexpr int kQpA = kRows * 128;          // [128 rows][64 slots] bf16, SW128
constexpr int kQpB = 2 * 64 * 128;         // [2 chunks][64 keys][64 dims], SW128
constexpr int kQpStage = kQpA + kQpB;      // 32 KB
constexpr int kQpOffSt = kQpStages * kQpStage;
constexpr int kQpOffBar = kQpOffSt + 4 * 2 * kQdStBytes;
constexpr int kQpNumBars = 2 * kQpStages + 4;
constexpr int kQpOffTmemPtr = kQpOffBar + 8 * kQpNumBars;
constexpr int kQpSmem = kQpOffTmemPtr + 16 + 1024;
static_assert(kQpSmem <= 232448, "smem");

__global__ void __launch_bounds__(256, 1) __cluster_dims__(2, 1, 1) bwd_dq_pair_kernel(const __grid_constant__ TcDqParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (sbase - sraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int prt = (p.rows + 2 * kRows - 1) / (2 * kRows);  // pair row tiles per batch entry
  const int ntiles = p.batch * prt * 3;
  const int cid = (int)(blockIdx.x >> 1), ncl = (int)(gridDim.x >> 1);
  struct Tile {
    int bi, r0, slice, lbq, se, nsc, nch;
  };
  auto decode = [&](int t) {
    Tile T;
    T.slice = t % 3;
    const int rest = t / 3;
    T.bi = rest / prt;
    T.r0 = (rest - T.bi * prt) * 2 * kRows;
    const int t0 = (int)(((uint64_t)(uint32_t)T.r0 * p.h_m) >> p.h_p), QB = (p.q_start + t0) / p.b;
    T.lbq = QB - p.l + 1 < p.s ? p.s : QB - p.l + 1;
    T.se = (QB + 1 < p.s ? QB + 1 : p.s) * p.b;  // sink slots the rows' block can see
    const int nl = QB >= T.lbq ? (QB + 1 - T.lbq) * p.b : 0;
    T.nsc = (T.se + 63) / 64;
    T.nch = T.nsc + nl / 64;
    return T;
  };
  auto chunk = [&](const Tile& T, int c, int& slot, int& key) {
    if (c < T.nsc) {
      slot = key = 64 * c;
    } else {
      const int i = 64 * (c - T.nsc);
      slot = p.s * p.b + i;
      key = T.lbq * p.b + i;
    }
  };
  // barriers: Full[kQpStages] (leader), Empty[kQpStages], AccFull[2], AccFree[2] (leader, 4 warps x 2 CTAs)
  auto bar = [&](int i) { return sbase + kQpOffBar + 8 * i; };
  const int kAccFull = 2 * kQpStages, kAccFree = kAccFull + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + kQpOffTmemPtr);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kQpStages; ++i) {
      mbar_init(bar(i), 1);
      mbar_init(bar(kQpStages + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kAccFull + i), 1);
      mbar_init(bar(kAccFree + i), 8);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.ds_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(&p.dq_map);
  }
  if (warp == 1) tmem_alloc<2>(smem_u32(tmem_ptr), 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  if (warp == 0) {
    // ---------------------------------------------------------------- TMA (each CTA: its rows, its dims)
    const uint64_t pol = policy_evict_normal(), pol_k = policy_evict_last();
    const uint32_t full_l = mapa(bar(0), 0);
    uint32_t slot = 0, ph = 0;
    for (int t = cid; t < ntiles; t += ncl) {
      const Tile T = decode(t);
      for (int c = 0; c < T.nch; ++c) {
        int sl, key;
        chunk(T, c, sl, key);
        mbar_wait(bar(kQpStages + slot), ph ^ 1);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(slot), 2 * kQpStage);
          const uint32_t dst = sbase + slot * kQpStage;
          tma_load_3d_pair(dst, &p.ds_map, sl, T.r0 + kRows * (int)rank, T.bi, full_l + 8 * slot, pol);
          tma_load_4d_pair(dst + kQpA, &p.k_map, 0, key, 4 * T.slice + 2 * (int)rank, T.bi, full_l + 8 * slot, pol_k);
        }
        __syncwarp();
        if (++slot == kQpStages) {
          slot = 0;
          ph ^= 1;
        }
      }
    }
    for (int i = 0; i < kQpStages; ++i) {  // drain: the last Empty commits land before this CTA exits
      mbar_wait(bar(kQpStages + slot), ph ^ 1);
      if (++slot == kQpStages) {
        slot = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- UMMA issuer (leader)
    if (rank == 0) {
      constexpr uint32_t id256 = idesc_bf16_f32(256, 256, false, true), id128 = idesc_bf16_f32(256, 128, false, true);
      uint32_t slot = 0, ph = 0;
      int n = 0;
      for (int t = cid; t < ntiles; t += ncl, ++n) {
        const Tile T = decode(t);
        const int ab = n & 1, use = n >> 1;
        mbar_wait(bar(kAccFree + ab), (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t id = T.slice < 2 ? id256 : id128;
        for (int c = 0; c < T.nch; ++c) {
          const int nk = c < T.nsc && T.se - 64 * c < 64 ? (T.se - 64 * c) / 16 : 4;
          mbar_wait(bar(slot), ph);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a = sbase + slot * kQpStage;
            for (int k = 0; k < nk; ++k)
              umma_bf16_pair(tmem + 256 * ab, sdesc_sw128(a + 32 * k, 16, 1024),
                             sdesc_sw128(a + kQpA + 2048 * k, 8192, 1024), id, (c | k) != 0);
            umma_commit_pair_mc(bar(kQpStages + slot), 3);
          }
          __syncwarp();
          if (++slot == kQpStages) {
            slot = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) umma_commit_pair_mc(bar(kAccFull + ab), 3);
        __syncwarp();
      }
      for (int u = n - 2 < 0 ? 0 : n - 2; u < n; ++u)  // the partner's last AccFree arrivals land before exit
        mbar_wait(bar(kAccFree + (u & 1)), (u >> 1) & 1);
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue (thread = row, TMA stores)
    const int q = warp - 4;
    const uint32_t st0 = sbase + kQpOffSt + (uint32_t)q * 2 * kQdStBytes, sw = (uint32_t)(lane & 7);
    const uint32_t afree0 = mapa(bar(kAccFree), 0);
    int n = 0, k = 0;
    for (int t = cid; t < ntiles; t += ncl, ++n) {
      const Tile T = decode(t);
      const int ab = n & 1, use = n >> 1;
      mbar_wait(bar(kAccFull + ab), use & 1);
      tc_fence_after();
      const int ng = T.slice < 2 ? 8 : 2;  // 32-dim groups stored (the third slice: dims 512..575)
      for (int g = 0; g < ng; ++g, ++k) {
        uint32_t v[32];
        if (T.nch > 0) {
          tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 256 * ab + 32 * g, v);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = 0u;
        }
        if (g == ng - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(afree0 + 8 * ab);
        }
        const uint32_t sb = st0 + (uint32_t)(k & 1) * kQdStBytes;
        if (lane == 0) bulk_wait_group_read1();
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 8; ++u)
          st_shared_v4(sb + lane * 128 + ((u ^ sw) << 4), __float_as_uint(__uint_as_float(v[4 * u]) * p.scale),
                       __float_as_uint(__uint_as_float(v[4 * u + 1]) * p.scale),
                       __float_as_uint(__uint_as_float(v[4 * u + 2]) * p.scale),
                       __float_as_uint(__uint_as_float(v[4 * u + 3]) * p.scale));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_3d(&p.dq_map, sb, 256 * T.slice + 32 * g, T.r0 + kRows * (int)rank + 32 * q, T.bi);
          bulk_commit_group();
        }
      }
    }
    if (lane == 0) bulk_wait_group0();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}

// D_r = dO_r . O_r (fp32), one warp per row (bf16 O and dO with o's strides, d_v 512)
__global__ void __launch_bounds__(256) bwd_D_kernel(const uint16_t* o, const uint16_t* dout, float* D, int32_t rows,
                                                   int32_t batch, int64_t o_sb, int64_t o_st, int64_t o_sh,
                                                   uint32_t h_m, uint32_t h_p, int32_t H) {
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= (int64_t)batch * rows) return;
  const int bi = (int)(gw / rows), r = (int)(gw - (int64_t)bi * rows);
  const int t = (int)(((uint64_t)(uint32_t)r * h_m) >> h_p), h = r - t * H;
  const int64_t off = bi * o_sb + (int64_t)t * o_st + (int64_t)h * o_sh;
  float acc = 0.f;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint4 ov = *reinterpret_cast<const uint4*>(o + off + 8 * (lane + 32 * u));
    const uint4 dv = *reinterpret_cast<const uint4*>(dout + off + 8 * (lane + 32 * u));
    const uint32_t oa[4] = {ov.x, ov.y, ov.z, ov.w}, da[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc = fmaf(__uint_as_float(oa[e] << 16), __uint_as_float(da[e] << 16), acc);
      acc = fmaf(__uint_as_float(oa[e] & 0xFFFF0000u), __uint_as_float(da[e] & 0xFFFF0000u), acc);
    }
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o2);
  if (lane == 0) D[gw] = acc;
}

}  // namespace

// Packed row layout (rows = tokens x heads at a uniform stride) for the 2-D row view of q and dO.
bool backward_tc_eligible(const AttnProblem& a, const void* dout) {
  (void)dout;
  return a.q_st == (int64_t)a.heads * a.q_sh && a.o_st == (int64_t)a.heads * a.o_sh && a.q_sh >= 576 &&
         a.o_sh >= 512;
}

cudaError_t launch_bwd_dkdv_tc(const AttnProblem& a, const void* dout, float* dk, float* dv, const float* D,
                               float* part, uint16_t* ds, int nsplit, int n_sink, cudaStream_t st) {
  TcBwdParams p;
  memset(&p, 0, sizeof(p));  // debug / pair-only fields default to off
  const auto& kv = a.kv.seg[0];
  const uint64_t rows = (uint64_t)a.n_q * a.heads;
  if (!encode_4d_chunks(&p.q_map, a.q, kDqk, rows, a.batch, a.q_sh, a.q_sb, kRows, 2) ||
      !encode_4d_chunks(&p.o_map, dout, kDv, rows, a.batch, a.o_sh, a.o_sb, kRows, 2) ||
      !encode_4d_chunks(&p.k_map, kv.k, kDqk, (uint64_t)a.n_kv, a.batch, kv.k_st, kv.k_sb, kKeys, 9))
    return cudaErrorInvalidValue;
  p.lse = a.lse;
  p.D = D;
  p.dk = dk;
  p.dv = dv;
  p.part = part;
  p.ds = ds;
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
  p.nsplit = nsplit;
  p.n_sink = n_sink;
  {
    uint32_t l = 0;
    while ((1ull << l) < (uint64_t)a.heads) ++l;
    p.h_p = 31 + l;
    p.h_m = (uint32_t)(((1ull << p.h_p) + a.heads - 1) / a.heads);
  }
  cudaError_t e = cudaFuncSetAttribute(bwd_dkdv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  if (e != cudaSuccess) return e;
  const int64_t kt = (a.n_kv + kKeys - 1) / kKeys;
  const int64_t nst = a.sparse && nsplit > 1 ? ((int64_t)a.s * a.b + kKeys - 1) / kKeys : 0;
  const int64_t ns = nst < kt ? nst : kt;  // sink tiles, split over rows
  bwd_dkdv_tc_kernel<<<(unsigned)(a.batch * (ns * nsplit + kt - ns)), 256, kSmem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool backward_pair_eligible(const AttnProblem& a) { return a.sparse && a.b == kPKeys; }

// Row splits of the pair key kernels. A sink tile is attended by every row, a local tile by <= l query blocks;
// both are cut into pieces of P whole query blocks, P the largest (up to l) whose clusters -- B x (sink tiles x
// ceil(NB / P) + local tiles x ceil(l / P)) -- fit the device's cluster slots: at 8K one piece per local tile
// (P = 7), at 2K P = 2. Split tiles write fp32 partials that a fixed-order reduce sums. Deterministic for a device.
PairSplits backward_pair_splits(const AttnProblem& a) {
  PairSplits r{1, 1};
  if (!backward_pair_eligible(a) || a.n_kv == 0 || a.batch == 0 || a.n_q == 0) return r;
  const int64_t kt = (a.n_kv + kPKeys - 1) / kPKeys;
  const int64_t nb = ((int64_t)a.q_start + a.n_q + a.b - 1) / a.b - a.q_start / a.b;  // query blocks
  const int64_t ns = a.s < kt ? a.s : kt;
  const int64_t slots = device_sm_count() / 2;
  int64_t P = a.l;
  for (int64_t c = a.l; c >= 1; --c) {
    const int64_t sn = a.s == 0 ? 1 : ((nb + c - 1) / c > 64 ? 64 : (nb + c - 1) / c);
    const int64_t ls = (a.l + c - 1) / c;
    if (a.batch * (ns * sn + (kt - ns) * ls) > slots) break;
    P = c;
  }
  r.nsplit = a.s == 0 ? 1 : (int)((nb + P - 1) / P > 64 ? 64 : (nb + P - 1) / P);
  r.lsplit = (int)((a.l + P - 1) / P);
  return r;
}
int backward_local_splits(const AttnProblem& a) { return backward_pair_splits(a).lsplit; }
size_t backward_local_part_bytes(const AttnProblem& a) {
  const PairSplits sp = backward_pair_splits(a);
  if (sp.lsplit <= 1) return 0;
  const int64_t kt = (a.n_kv + kPKeys - 1) / kPKeys;
  const int64_t ns = a.s < kt ? a.s : kt;
  if (kt - ns <= 0) return 0;
  return sizeof(float) * (size_t)a.batch * (kt - ns) * sp.lsplit * kPKeys * kDkv;
}

// 64-key tiles (two kernels, dV then dK): the tile must lie in one block (b % 64 == 0) when sparse
bool backward_key64_eligible(const AttnProblem& a) { return !a.sparse || a.b % k64Keys == 0; }

unsigned long long* g_bwd_trace = nullptr;  // loza_debug_set_bwd_trace
int g_bwd_trace_cluster = 0, g_bwd_trace_mode = 0;

// 128-key CTA-pair kernels (dV, then dK reading P back from the dS row buffer): SSA with b == 128
static cudaError_t launch_bwd_pair_tc(const AttnProblem& a, const void* dout, float* dk, float* dv, const float* D,
                                      float* part, float* part_local, uint16_t* ds, int nsplit, int n_sink,
                                      cudaStream_t st, cudaEvent_t d_ready) {
  TcBwdParams p;
  memset(&p, 0, sizeof(p));  // debug / pair-only fields default to off
  const auto& kv = a.kv.seg[0];
  const uint64_t rows = (uint64_t)a.n_q * a.heads;
  TcBwdParams pk;  // the dK kernel's: its K tile is V's 8 chunks
  if (!encode_4d_chunks(&p.q_map, a.q, kDqk, rows, a.batch, a.q_sh, a.q_sb, kRows, 2) ||
      !encode_4d_chunks(&p.o_map, dout, kDv, rows, a.batch, a.o_sh, a.o_sb, kRows, 2) ||
      !encode_4d_chunks(&p.k_map, kv.k, kDqk, (uint64_t)a.n_kv, a.batch, kv.k_st, kv.k_sb, 64, 9) ||
      !encode_4d_chunks(&pk.k_map, kv.k, kDqk, (uint64_t)a.n_kv, a.batch, kv.k_st, kv.k_sb, 64, 8) ||
      !encode_4d_chunks(&p.q4_map, a.q, kDqk, rows, a.batch, a.q_sh, a.q_sb, kPHalf, 4) ||
      !encode_4d_chunks(&p.q1_map, a.q, kDqk, rows, a.batch, a.q_sh, a.q_sb, kPHalf, 1) ||
      !encode_4d_chunks(&p.o4_map, dout, kDv, rows, a.batch, a.o_sh, a.o_sb, kPHalf, 4))
    return cudaErrorInvalidValue;
  p.lse = a.lse;
  p.D = D;
  p.dk = dk;
  p.dv = dv;
  p.part = part;
  p.ds = ds;
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
  p.nsplit = nsplit;
  p.n_sink = n_sink;
  {
    uint32_t l = 0;
    while ((1ull << l) < (uint64_t)a.heads) ++l;
    p.h_p = 31 + l;
    p.h_m = (uint32_t)(((1ull << p.h_p) + a.heads - 1) / a.heads);
  }
  p.trace = g_bwd_trace_mode == kPairDv ? g_bwd_trace : nullptr;
  p.trace_cluster = g_bwd_trace_cluster;
  const CUtensorMap k8 = pk.k_map;
  pk = p;
  pk.k_map = k8;
  pk.trace = g_bwd_trace_mode == kPairDk ? g_bwd_trace : nullptr;
  {  // the dS row buffer as TMA store target: {W slots, rows, B}, box {64 slots, 128 rows, 1}, SW128
    const int W = (a.s + a.l) * a.b;
    if (!encode_3d(&p.ds_map, ds, (uint64_t)W, rows, a.batch, W, (int64_t)rows * W, kRows)) return cudaErrorInvalidValue;
    pk.ds_map = p.ds_map;
  }
  // the dK kernel's q1 box: [1 chunk][128 rows] (dK^T's third dim group)
  if (!encode_4d_chunks(&pk.q1_map, a.q, kDqk, rows, a.batch, a.q_sh, a.q_sb, kRows, 1)) return cudaErrorInvalidValue;
  const int64_t kt = (a.n_kv + kPKeys - 1) / kPKeys;
  const int64_t ns = a.s < kt ? a.s : kt;  // sink tiles (nsplit clusters each), then the local tiles (ls each)
  const int ls = backward_local_splits(a);
  p.lsplit = pk.lsplit = ls;
  p.part_local = pk.part_local = ls > 1 ? part_local : nullptr;
  if (ls > 1 && kt > ns && !part_local) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)(2 * a.batch * (ns * nsplit + (kt - ns) * ls)));
  cudaError_t e = cudaFuncSetAttribute(bwd_pair_tc_kernel<kPairDv>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       PairCfg<kPairDv>::kSmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bwd_pair_tc_kernel<kPairDk>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PairCfg<kPairDk>::kSmem);
  if (e != cudaSuccess) return e;
  bwd_pair_tc_kernel<kPairDv><<<grid, kPThreads, PairCfg<kPairDv>::kSmem, st>>>(p);
  count_launch();
  if (d_ready && (e = cudaStreamWaitEvent(st, d_ready, 0)) != cudaSuccess) return e;  // D (side stream) for dS
  bwd_pair_tc_kernel<kPairDk><<<grid, kPThreads, PairCfg<kPairDk>::kSmem, st>>>(pk);
  count_launch();
  if (ls > 1 && kt > ns) {
    const int64_t n = (int64_t)a.batch * (kt - ns) * kPKeys * (kDkv / 4);
    bwd_local_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part_local, dk, dv, a.batch, (int32_t)a.n_kv,
                                                                         (int32_t)ns, (int32_t)(kt - ns), ls);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_bwd_key64_tc(const AttnProblem& a, const void* dout, float* dk, float* dv, const float* D,
                                float* part, uint16_t* ds, int nsplit, int n_sink, cudaStream_t st,
                                cudaEvent_t d_ready, bool allow_pair, float* part_local) {
  if (allow_pair && ds && backward_pair_eligible(a))
    return launch_bwd_pair_tc(a, dout, dk, dv, D, part, part_local, ds, nsplit, n_sink, st, d_ready);
  TcBwdParams p;
  memset(&p, 0, sizeof(p));  // debug / pair-only fields default to off
  const auto& kv = a.kv.seg[0];
  const uint64_t rows = (uint64_t)a.n_q * a.heads;
  if (!encode_4d_chunks(&p.q_map, a.q, kDqk, rows, a.batch, a.q_sh, a.q_sb, kRows, 2) ||
      !encode_4d_chunks(&p.o_map, dout, kDv, rows, a.batch, a.o_sh, a.o_sb, kRows, 2) ||
      !encode_4d_chunks(&p.k_map, kv.k, kDqk, (uint64_t)a.n_kv, a.batch, kv.k_st, kv.k_sb, k64Keys, 9))
    return cudaErrorInvalidValue;
  p.lse = a.lse;
  p.D = D;
  p.dk = dk;
  p.dv = dv;
  p.part = part;
  p.ds = ds;
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
  p.nsplit = nsplit;
  p.n_sink = n_sink;
  {
    uint32_t l = 0;
    while ((1ull << l) < (uint64_t)a.heads) ++l;
    p.h_p = 31 + l;
    p.h_m = (uint32_t)(((1ull << p.h_p) + a.heads - 1) / a.heads);
  }
  const int64_t kt = (a.n_kv + k64Keys - 1) / k64Keys;
  const int64_t nst = a.sparse && nsplit > 1 ? ((int64_t)a.s * a.b + k64Keys - 1) / k64Keys : 0;
  const int64_t ns = nst < kt ? nst : kt;  // sink tiles, split over rows
  const dim3 grid((unsigned)(a.batch * (ns * nsplit + kt - ns)));
  cudaError_t e = cudaFuncSetAttribute(bwd_key64_tc_kernel<kDvOnly>, cudaFuncAttributeMaxDynamicSharedMemorySize, k64Smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bwd_key64_tc_kernel<kDkOnly>, cudaFuncAttributeMaxDynamicSharedMemorySize, k64Smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(bwd_key64_tc_kernel<kDkFromP>, cudaFuncAttributeMaxDynamicSharedMemorySize, k64Smem);
  if (e != cudaSuccess) return e;
  // with the dS row buffer (SSA): the dV kernel leaves P there and the dK kernel reads it (no S recompute)
  bwd_key64_tc_kernel<kDvOnly><<<grid, 256, k64Smem, st>>>(p);
  count_launch();
  if (d_ready && (e = cudaStreamWaitEvent(st, d_ready, 0)) != cudaSuccess) return e;  // D (side stream) for dS
  if (ds)
    bwd_key64_tc_kernel<kDkFromP><<<grid, 256, k64Smem, st>>>(p);
  else
    bwd_key64_tc_kernel<kDkOnly><<<grid, 256, k64Smem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

// dS-buffer path (SSA): rows of a 128-row tile must share one query block
bool backward_ds_eligible(const AttnProblem& a) {
  if (!a.sparse) return false;
  const int H = a.heads;
  return a.causal && (H % kRows == 0 || (kRows % H == 0 && kRows / H <= 32 && a.b % (kRows / H) == 0));
}
size_t backward_ds_bytes(const AttnProblem& a) {
  if (!a.sparse) return 0;
  return (size_t)2 * a.batch * a.n_q * a.heads * ((size_t)(a.s + a.l) * a.b);
}

cudaError_t launch_bwd_D(const AttnProblem& a, const void* dout, float* D, cudaStream_t st) {
  const int64_t rows = (int64_t)a.n_q * a.heads, warps = rows * a.batch;
  uint32_t l = 0;
  while ((1ull << l) < (uint64_t)a.heads) ++l;
  const uint32_t hp = 31 + l, hm = (uint32_t)(((1ull << hp) + a.heads - 1) / a.heads);
  bwd_D_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(static_cast<const uint16_t*>(a.o),
                                                             static_cast<const uint16_t*>(dout), D, (int32_t)rows,
                                                             a.batch, a.o_sb, a.o_st, a.o_sh, hm, hp, a.heads);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_bwd_dq_tc(const AttnProblem& a, const uint16_t* ds, float* dq, cudaStream_t st, bool pair_keys) {
  TcDqParams p;
  memset(&p, 0, sizeof(p));
  const auto& kv = a.kv.seg[0];
  const int W = (a.s + a.l) * a.b;
  const uint64_t rows = (uint64_t)a.n_q * a.heads;
  // the pair GEMM needs every slot of a row's visible blocks written (the 128-key pair key kernels) and 256-row
  // tiles inside one query block
  const bool pair = pair_keys && ((int64_t)a.b * a.heads) % (2 * kRows) == 0;
  if (!encode_3d(&p.ds_map, ds, (uint64_t)W, rows, a.batch, W, (int64_t)rows * W, kRows) ||
      !encode_4d_chunks(&p.k_map, kv.k, kDqk, (uint64_t)a.n_kv, a.batch, kv.k_st, kv.k_sb, 64, pair ? 2 : 3) ||
      !encode_3d_f32(&p.dq_map, dq, kDqk, rows, a.batch, kDqk, (int64_t)rows * kDqk, 32))
    return cudaErrorInvalidValue;
  p.dq = dq;
  p.rows = (int32_t)rows;
  p.heads = a.heads;
  p.n_kv = (int32_t)a.n_kv;
  p.q_start = (int32_t)a.q_start;
  p.s = a.s;
  p.l = a.l;
  p.b = a.b;
  p.kv32 = (int32_t)((a.n_kv + 31) / 32 * 32);
  p.batch = a.batch;
  p.scale = a.scale;
  {
    uint32_t l = 0;
    while ((1ull << l) < (uint64_t)a.heads) ++l;
    p.h_p = 31 + l;
    p.h_m = (uint32_t)(((1ull << p.h_p) + a.heads - 1) / a.heads);
  }
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaError_t e;
  if (pair) {
    if ((e = cudaFuncSetAttribute(bwd_dq_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kQpSmem)) !=
        cudaSuccess)
      return e;
    const int64_t prt = ((int64_t)rows + 2 * kRows - 1) / (2 * kRows), tiles = a.batch * prt * 3;
    const int64_t ncl = tiles < sms / 2 ? tiles : sms / 2;
    bwd_dq_pair_kernel<<<(unsigned)(2 * ncl), 256, kQpSmem, st>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  e = cudaFuncSetAttribute(bwd_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kQdSmem);
  if (e != cudaSuccess) return e;
  const int64_t rt = ((int64_t)rows + kRows - 1) / kRows, tiles = a.batch * rt * 3;
  bwd_dq_tc_kernel<<<(unsigned)(tiles < sms ? tiles : sms), 256, kQdSmem, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza

// debug hook (not part of include/loza.h): clock64 timeline of pair cluster `cluster` of the backward pair
// kernel `mode` (1 dV, 2 dK) into dev_ptr (tools/trace_bwd.py)
extern "C" void loza_debug_set_bwd_trace(void* dev_ptr, int32_t cluster, int32_t mode) {
  loza::g_bwd_trace = (unsigned long long*)dev_ptr;
  loza::g_bwd_trace_cluster = cluster;
  loza::g_bwd_trace_mode = mode;
}
