// tcgen05 bf16 attention prefill over the absorbed latent MLA KV (d_qk 576, d_v 512):
// SSA (Eq. 4) and the full-attention comparator (Eq. 1).
//
// Design:
//  * CTA pair (cluster of 2, cta_group::2). One work unit = 128 consecutive query
//    rows of the [n_q*H] row space (H=64: two tokens x 64 heads), CTA r owns rows
//    64r..64r+63. Units never straddle a query block (H*b % 128 == 0), so every
//    row of a unit has the same selected key blocks: the block list is the closed
//    form of the integer prologue (select_blocks.cu), computed in-kernel.
//  * Per 128-key tile: S = Q K^T via 36 UMMAs M=128 N=128 K=16 (A = resident Q,
//    B = K half per CTA), S into TMEM (double buffered, 64 cols each in the 2x2
//    fold); online softmax in registers (row max exchanged between the two
//    TMEM lanes that hold a row's two key halves); P (bf16) to SMEM; O += P V
//    via 16 UMMAs M=128 N=256 K=16 (B = V, MN-major) into a 64x512 fp32 TMEM
//    accumulator per CTA (256 cols). TMEM: O 256 + S 2x64 of 512 columns.
//  * Loads: TMA (SWIZZLE_128B) into a ring of 8 KB stages shared by K chunks
//    (64 keys x 64 dims) and V slabs (32 keys x 128 dims); both CTAs' loads
//    complete on the leader's barrier; one elected thread of the leader issues
//    every MMA; commits are multicast to both CTAs.
//  * FA-style pipelining: MMA order S(0), S(1), PV(0), S(2), PV(1), ... so the
//    softmax of tile t overlaps PV(t-1) and S(t+1). Lazy rescaling: O and l are
//    rescaled only when a row max grows by more than 2^8 (exact: the final
//    normalisation uses the same stale max).
//  * Persistent: grid = min(#units, SMs/2) clusters, units in reverse order
//    (heaviest causal rows first).
#include <math.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {
using namespace sm100;

constexpr int kDqk = 576, kDv = 512, kChunks = 9;
constexpr int kThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 softmax/epilogue
constexpr int kStageBytes = 8192;
constexpr int kStages = 14;
constexpr int kQBytes = kChunks * 64 * 128;  // 73728 per CTA
constexpr int kPBytes = 2 * 64 * 128;        // 16384 per buffer (2 key chunks x 64 rows)
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffRing = kOffP + 2 * kPBytes;
constexpr int kOffBar = kOffRing + kStages * kStageBytes;
// barrier block
constexpr int kBarRingFull = 0;
constexpr int kBarRingEmpty = kBarRingFull + kStages;
constexpr int kBarQFull = kBarRingEmpty + kStages;
constexpr int kBarQEmpty = kBarQFull + 1;
constexpr int kBarSFull = kBarQEmpty + 1;   // [2]
constexpr int kBarSFree = kBarSFull + 2;    // [2]
constexpr int kBarPFull = kBarSFree + 2;    // [2]
constexpr int kBarOFull = kBarPFull + 2;    // [2]
constexpr int kBarOFree = kBarOFull + 2;
constexpr int kNumBars = kBarOFree + 1;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffRed = (kOffTmemPtr + 4 + 15) & ~15;  // float [2 buf][2 half][64]
constexpr int kOffLsum = kOffRed + 2 * 2 * 64 * 4;     // float [2 half][64]
constexpr int kSmemUsed = kOffLsum + 2 * 64 * 4;
constexpr int kSmemAlloc = kSmemUsed + 1024;  // + alignment slack
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 0, kTmemS = 256;
constexpr uint32_t kSoftmaxWarps = 4;
constexpr uint32_t kArrivalsPerPair = 2 * kSoftmaxWarps;  // softmax warps of both CTAs

struct PrefillParams {
  CUtensorMap q_map;
  CUtensorMap k_map[3];
  CUtensorMap v_map[3];
  int64_t seg_begin[3];
  int32_t nseg;
  int32_t batch, n_q, heads;
  int64_t q_start, n_kv;
  int32_t s, l, b, sparse, causal;
  float scale_log2;
  void* o;
  int64_t o_sb;
  int32_t out_bf16;
  float* lse;
  int64_t units_per_batch, total_units;
};

struct Unit {
  int32_t bi;
  int64_t row0;          // first row of the unit in the batch's [n_q*H] rows
  int64_t tok_lo, tok_hi;  // absolute positions
  int32_t n_sink, loc_begin, n_tiles;  // tiles of 128 keys
};

__device__ __forceinline__ Unit make_unit(const PrefillParams& p, int64_t u) {
  Unit U;
  U.bi = (int32_t)(u / p.units_per_batch);
  U.row0 = (u % p.units_per_batch) * 128;
  const int64_t rows = (int64_t)p.n_q * p.heads;
  int64_t rlast = U.row0 + 127;
  if (rlast > rows - 1) rlast = rows - 1;
  U.tok_lo = p.q_start + U.row0 / p.heads;
  U.tok_hi = p.q_start + rlast / p.heads;
  const int64_t last_tile = p.causal ? U.tok_hi / 128 : (p.n_kv - 1) / 128;
  if (!p.sparse) {
    U.n_sink = 0;
    U.loc_begin = 0;
    U.n_tiles = (int32_t)(last_tile + 1);
    return U;
  }
  const int64_t tpb = p.b / 128, QB = U.tok_lo / p.b;
  int64_t sink_end = (QB + 1 < p.s ? QB + 1 : p.s) * tpb;
  if (sink_end > last_tile + 1) sink_end = last_tile + 1;
  int64_t lb = QB - p.l + 1;
  if (lb < p.s) lb = p.s;
  lb *= tpb;
  int64_t le = (QB + 1) * tpb;
  if (le > last_tile + 1) le = last_tile + 1;
  U.n_sink = (int32_t)sink_end;
  U.loc_begin = (int32_t)lb;
  U.n_tiles = (int32_t)(sink_end + (le > lb ? le - lb : 0));
  return U;
}
__device__ __forceinline__ int64_t tile_k0(const Unit& U, int i) {
  return (int64_t)(i < U.n_sink ? i : U.loc_begin + (i - U.n_sink)) * 128;
}
__device__ __forceinline__ int seg_of(const PrefillParams& p, int64_t k0) {
  int s = 0;
  if (p.nseg > 1 && k0 >= p.seg_begin[1]) s = 1;
  if (p.nseg > 2 && k0 >= p.seg_begin[2]) s = 2;
  return s;
}
__device__ __forceinline__ int64_t unit_index(const PrefillParams& p, int64_t it) {
  return p.total_units - 1 - it;  // heaviest (latest rows) first
}

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    prefill_tc_kernel(const __grid_constant__ PrefillParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  float* lsum = reinterpret_cast<float*>(smem + kOffLsum);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar(kBarRingFull + i), 1);
      mbar_init(bar(kBarRingEmpty + i), 1);
    }
    mbar_init(bar(kBarQFull), 1);
    mbar_init(bar(kBarQEmpty), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), kArrivalsPerPair);
      mbar_init(bar(kBarPFull + i), kArrivalsPerPair);
      mbar_init(bar(kBarOFull + i), 1);
    }
    mbar_init(bar(kBarOFree), kArrivalsPerPair);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    for (int i = 0; i < p.nseg; ++i) {
      prefetch_tmap(&p.k_map[i]);
      prefetch_tmap(&p.v_map[i]);
    }
  }
  if (warp == 1) tmem_alloc<2>(smem_u32(tmem_ptr_smem), kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;

  const int64_t n_iter_total = p.total_units;
  const int64_t ncl = nclusters_x();
  const int64_t cid = cluster_id_x();

  if (warp == 0) {
    // ===================================================== TMA producer (both CTAs)
    if (lane == 0) {
      const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
      uint32_t stage = 0, phase = 0, uc = 0;
      auto next = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      };
      auto acquire = [&]() -> uint32_t {
        mbar_wait(bar(kBarRingEmpty + stage), phase ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(bar(kBarRingFull + stage), 2 * kStageBytes);
        return sbase + kOffRing + stage * kStageBytes;
      };
      auto load_k = [&](const Unit& U, int64_t k0) {
        const int sg = seg_of(p, k0);
        const int32_t row = (int32_t)(k0 - p.seg_begin[sg]) + 64 * (int32_t)rank;
        for (int c = 0; c < kChunks; ++c) {
          const uint32_t dst = acquire();
          tma_load_3d_pair(dst, &p.k_map[sg], c * 64, row, U.bi, mapa(bar(kBarRingFull + stage), 0), pol_kv);
          next();
        }
      };
      auto load_v = [&](const Unit& U, int64_t k0) {
        const int sg = seg_of(p, k0);
        const int32_t row = (int32_t)(k0 - p.seg_begin[sg]);
        for (int kq = 0; kq < 4; ++kq)
          for (int nh = 0; nh < 2; ++nh) {
            const uint32_t dst = acquire();
            const uint32_t fb = mapa(bar(kBarRingFull + stage), 0);
            for (int e = 0; e < 2; ++e)
              tma_load_3d_pair(dst + e * 4096, &p.v_map[sg], 256 * nh + 128 * (int)rank + 64 * e, row + 32 * kq,
                               U.bi, fb, pol_kv);
            next();
          }
      };
      for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
        const Unit U = make_unit(p, unit_index(p, it));
        mbar_wait(bar(kBarQEmpty), (uc & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(bar(kBarQFull), 2 * kQBytes);
        const uint32_t qfb = mapa(bar(kBarQFull), 0);
        for (int c = 0; c < kChunks; ++c)
          tma_load_3d_pair(sbase + kOffQ + c * 8192, &p.q_map, c * 64, (int32_t)(U.row0 + 64 * rank), U.bi, qfb,
                           pol_q);
        load_k(U, tile_k0(U, 0));
        for (int i = 1; i < U.n_tiles; ++i) {
          load_k(U, tile_k0(U, i));
          load_v(U, tile_k0(U, i - 1));
        }
        load_v(U, tile_k0(U, U.n_tiles - 1));
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer (leader CTA only)
    if (rank == 0 && lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 256, false, true);
      uint32_t stage = 0, phase = 0, uc = 0;
      uint32_t g = 0;
      auto next = [&]() {
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      };
      auto issue_s = [&](uint32_t gi) {
        const uint32_t buf = gi & 1;
        mbar_wait(bar(kBarSFree + buf), ((gi >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + kTmemS + 64 * buf;
        for (int c = 0; c < kChunks; ++c) {
          mbar_wait(bar(kBarRingFull + stage), phase);
          tc_fence_after();
          const uint32_t a0 = sbase + kOffQ + c * 8192, b0 = sbase + kOffRing + stage * kStageBytes;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_pair(d, sdesc_sw128(a0 + 32 * k, 16, 1024), sdesc_sw128(b0 + 32 * k, 16, 1024), idesc_s,
                           (c | k) != 0);
          umma_commit_pair_mc(bar(kBarRingEmpty + stage), 3);
          next();
        }
        umma_commit_pair_mc(bar(kBarSFull + buf), 3);
      };
      auto issue_pv = [&](uint32_t gi, bool first) {
        const uint32_t buf = gi & 1;
        mbar_wait(bar(kBarPFull + buf), (gi >> 1) & 1);
        if (first && uc > 0) mbar_wait(bar(kBarOFree), (uc - 1) & 1);
        tc_fence_after();
        const uint32_t pbase = sbase + kOffP + buf * kPBytes;
        for (int kq = 0; kq < 4; ++kq)
          for (int nh = 0; nh < 2; ++nh) {
            mbar_wait(bar(kBarRingFull + stage), phase);
            tc_fence_after();
            const uint32_t b0 = sbase + kOffRing + stage * kStageBytes;
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const uint32_t a = pbase + (kq >> 1) * 8192 + (kq & 1) * 64 + kk * 32;
              umma_bf16_pair(tmem + kTmemO + 128 * nh, sdesc_sw128(a, 16, 1024),
                             sdesc_sw128(b0 + kk * 2048, 4096, 1024), idesc_pv, !(first && kq == 0 && kk == 0));
            }
            umma_commit_pair_mc(bar(kBarRingEmpty + stage), 3);
            next();
          }
        umma_commit_pair_mc(bar(kBarOFull + buf), 3);
      };
      for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
        const Unit U = make_unit(p, unit_index(p, it));
        mbar_wait(bar(kBarQFull), uc & 1);
        tc_fence_after();
        const uint32_t g0 = g;
        for (int i = 0; i < U.n_tiles; ++i) {
          issue_s(g0 + i);
          if (i == U.n_tiles - 1) umma_commit_pair_mc(bar(kBarQEmpty), 3);
          if (i >= 1) issue_pv(g0 + i - 1, i - 1 == 0);
        }
        issue_pv(g0 + U.n_tiles - 1, U.n_tiles == 1);
        g += U.n_tiles;
      }
    }
  } else {
    // ===================================================== softmax + epilogue (warps 2..5, both CTAs)
    const uint32_t wq = warp & 3;
    const uint32_t tl = wq * 32 + lane;  // TMEM lane of this thread
    const uint32_t r = tl & 63, kh = tl >> 6;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const uint32_t sfree0 = mapa(bar(kBarSFree), 0), pfull0 = mapa(bar(kBarPFull), 0), ofree = mapa(bar(kBarOFree), 0);
    const float ln2 = 0.69314718055994531f;
    const int64_t rows_b = (int64_t)p.n_q * p.heads;
    const float sl2 = p.scale_log2;
    const int causal = p.causal;
    const int64_t n_kv = p.n_kv;
    uint32_t g = 0, uc = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = make_unit(p, unit_index(p, it));
      const int64_t row_g = U.row0 + 64 * rank + r;
      const bool row_ok = row_g < rows_b;
      const int64_t my_tok = p.q_start + (row_ok ? row_g : rows_b - 1) / p.heads;
      float m_used = -INFINITY, lrow = 0.f;
      for (int i = 0; i < U.n_tiles; ++i) {
        const uint32_t gi = g + i, buf = gi & 1;
        const int64_t k0 = tile_k0(U, i);
        const bool need_mask = (causal && k0 + 127 > U.tok_lo) || (k0 + 128 > n_kv);
        mbar_wait(bar(kBarSFull + buf), (gi >> 1) & 1);
        tc_fence_after();
        uint32_t sr[64];
        {
          uint32_t (&lo)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sr[0]);
          uint32_t (&hi)[32] = *reinterpret_cast<uint32_t(*)[32]>(&sr[32]);
          tmem_ld32(taddr + kTmemS + 64 * buf, lo);
          tmem_ld32(taddr + kTmemS + 64 * buf + 32, hi);
          tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(sfree0 + 8 * buf);
        float x[64];
        float tmax = -INFINITY;
        const int64_t kbase = k0 + 64 * kh;
#pragma unroll
        for (int j = 0; j < 64; ++j) {
          float v = __uint_as_float(sr[j]) * sl2;
          if (need_mask) {
            const int64_t kp = kbase + j;
            if ((causal && kp > my_tok) || kp >= n_kv) v = -INFINITY;
          }
          x[j] = v;
          tmax = fmaxf(tmax, v);
        }
        red[(buf * 2 + kh) * 64 + r] = tmax;
        named_bar_sync(1, 128);
        tmax = fmaxf(tmax, red[(buf * 2 + (kh ^ 1)) * 64 + r]);
        const bool resc = tmax > m_used + 8.0f;
        const float m_new = resc ? tmax : m_used;
        const float corr = resc ? ex2(m_used - m_new) : 1.0f;
        uint32_t pk[32];
        float psum = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float p0 = ex2(x[2 * j] - m_new), p1 = ex2(x[2 * j + 1] - m_new);
          pk[j] = pack_bf16x2(p0, p1);
          psum += __uint_as_float(pk[j] << 16) + __uint_as_float(pk[j] & 0xFFFF0000u);
        }
        if (i > 0) {
          const uint32_t gp = gi - 1;
          mbar_wait(bar(kBarOFull + (gp & 1)), (gp >> 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, resc)) {
#pragma unroll 1
            for (int c = 0; c < 8; ++c) {
              uint32_t ov[32];
              tmem_ld32(taddr + kTmemO + 32 * c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
              tmem_st32(taddr + kTmemO + 32 * c, ov);
            }
            tmem_wait_st();
          }
        }
        lrow = lrow * corr + psum;
        m_used = m_new;
        // P chunk kh, row r, 128-byte swizzled row
        const uint32_t prow = sbase + kOffP + buf * kPBytes + kh * 8192 + r * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          st_shared_v4(prow + ((u ^ (r & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(pfull0 + 8 * buf);
      }
      // ---------------- epilogue: O / l -> global
      const uint32_t gl = g + U.n_tiles - 1;
      mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
      tc_fence_after();
      lsum[kh * 64 + r] = lrow;
      named_bar_sync(1, 128);
      const float ltot = lrow + lsum[(kh ^ 1) * 64 + r];
      const float inv = 1.0f / ltot;
      char* obase = reinterpret_cast<char*>(p.o) +
                    ((int64_t)U.bi * p.o_sb + (row_ok ? row_g : 0) * kDv) * (p.out_bf16 ? 2 : 4);
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t ov[32];
        tmem_ld32(taddr + kTmemO + 32 * c, ov);
        tmem_wait_ld();
        const int nh = c >> 2, cc = c & 3;
        const int dim0 = 256 * nh + 128 * (int)kh + 32 * cc;
        if (row_ok) {
          if (p.out_bf16) {
            uint32_t w[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              w[j] = pack_bf16x2(__uint_as_float(ov[2 * j]) * inv, __uint_as_float(ov[2 * j + 1]) * inv);
            char* dst = obase + dim0 * 2;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) st_global_v4(dst + 16 * q4, w[4 * q4], w[4 * q4 + 1], w[4 * q4 + 2], w[4 * q4 + 3]);
          } else {
            char* dst = obase + dim0 * 4;
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4)
              st_global_v4(dst + 16 * q4, __float_as_uint(__uint_as_float(ov[4 * q4]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q4 + 1]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q4 + 2]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q4 + 3]) * inv));
          }
        }
      }
      if (p.lse && row_ok && kh == 0) {
        const int64_t h = row_g % p.heads, tl_ = row_g / p.heads;
        p.lse[((int64_t)U.bi * p.heads + h) * p.n_q + tl_] = (m_used + __log2f(ltot)) * ln2;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ofree);
      g += U.n_tiles;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, kTmemCols);
  }
}

}  // namespace

cudaError_t launch_prefill_tc(const AttnProblem& a, cudaStream_t st) {
  PrefillParams p;
  memset(&p, 0, sizeof(p));
  p.batch = a.batch;
  p.n_q = a.n_q;
  p.heads = a.heads;
  p.q_start = a.q_start;
  p.n_kv = a.n_kv;
  p.s = a.s;
  p.l = a.l;
  p.b = a.sparse ? a.b : 128;
  p.sparse = a.sparse;
  p.causal = a.causal;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.o = a.o;
  p.o_sb = a.o_sb;
  p.out_bf16 = a.out_bf16;
  p.lse = a.lse;
  const int64_t rows = (int64_t)a.n_q * a.heads;
  p.units_per_batch = (rows + 127) / 128;
  p.total_units = p.units_per_batch * a.batch;
  if (p.total_units == 0) return cudaSuccess;
  if (!encode_3d(&p.q_map, a.q, kDqk, rows, a.batch, kDqk, a.q_sb, 64)) return cudaErrorInvalidValue;
  p.nseg = a.kv.nseg;
  for (int i = 0; i < a.kv.nseg; ++i) {
    const KvSeg& s = a.kv.seg[i];
    p.seg_begin[i] = s.pos_begin;
    const uint64_t len = (uint64_t)(s.pos_end - s.pos_begin);
    if (!encode_3d(&p.k_map[i], s.k, kDqk, len, a.batch, s.k_st, s.k_sb, 64)) return cudaErrorInvalidValue;
    if (!encode_3d(&p.v_map[i], s.v, kDv, len, a.batch, s.v_st, s.v_sb, 32)) return cudaErrorInvalidValue;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int sms = device_sm_count();
  int64_t ncl = sms / 2;
  if (ncl > p.total_units) ncl = p.total_units;
  prefill_tc_kernel<<<(unsigned)(2 * ncl), kThreads, kSmemAlloc, st>>>(p);
  count_launch();
  return cudaGetLastError();
}


}  // namespace loza
