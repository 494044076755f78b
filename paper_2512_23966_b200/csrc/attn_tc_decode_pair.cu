// SSA decode with a CTA pair per sequence (Eq. 4 at p = seq_len - 1).
//
// The window of a sequence is at most (s+l)*b keys (8 tiles of 128 at (1,7,128)), read from HBM
// once per step whatever the context length. One cluster of 2 CTAs per sequence: CTA r owns heads
// [32 r, 32 r + 32), both CTAs consume every tile of the window, and every K / V stage is fetched
// ONCE from HBM with TMA multicast (each CTA loads half of the stage into both CTAs' shared memory).
// So the window is streamed at the pair's share of HBM bandwidth, no partial results exist and
// nothing needs merging (the split-KV alternative spent most of its time combining partials).
//
// Per CTA, per 128-key tile (transposed products keep M = 128, full-rate UMMA rows):
//   S^T[key][head]  = K Q^T   : UMMA M=128 (keys, A = K stage) N=32 (heads, B = Q chunk)   36 x K16
//   O^T[dim][head] += V^T P   : UMMA M=128 (dims, A = V stage, MN-major) N=32 (B = P, MN-major SW64)
// TMEM: O^T 4 groups x 32 columns, S^T 2 buffers x 32 columns. The softmax thread of TMEM lane k owns
// key k of the tile for the CTA's 32 heads; per-head maxima over keys use redux.sync.max.f32 within a
// warp and shared memory across the 4 key quarters; lazy rescaling (threshold 2^8) as in the prefill.
// Epilogue: O^T / l transposed through shared memory, then 16-byte coalesced stores.
#include <math.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {
using namespace sm100;

constexpr int kDqk = 576, kDv = 512, kChunks = 9, kH = 64, kHC = 32;  // heads per CTA
constexpr int kThreads = 192;  // warp 0 TMA, warp 1 UMMA, warps 2-5 softmax / epilogue
constexpr int kStageBytes = 16384;
constexpr int kStages = 10;
constexpr int kQBytes = kChunks * kHC * 128;  // 36864
constexpr int kPBytes = 128 * kHC * 2;        // 8192 per buffer: [128 keys][32 heads] bf16, SW64
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffRing = kOffP + 2 * kPBytes;
constexpr int kOffBar = kOffRing + kStages * kStageBytes;
constexpr int kBarFull = 0;
constexpr int kBarEmpty = kBarFull + kStages;
constexpr int kBarQFull = kBarEmpty + kStages;
constexpr int kBarSFull = kBarQFull + 1;  // [2]
constexpr int kBarSFree = kBarSFull + 2;  // [2]
constexpr int kBarPFull = kBarSFree + 2;  // [2]
constexpr int kBarOFull = kBarPFull + 2;  // [2]
constexpr int kNumBars = kBarOFull + 2;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffRed = (kOffTmemPtr + 4 + 15) & ~15;  // float [2 buf][4 quarters][32 heads]
constexpr int kSmemUsed = kOffRed + 2 * 4 * kHC * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kTmemS = 128;  // S^T buffer b at 128 + 32 b; O^T group g at 32 g
constexpr uint32_t kSmWarps = 4;

struct PairParams {
  CUtensorMap q_map, k_map, v_map;
  const int32_t* seq_lens;
  int32_t batch, s, l, b;
  int64_t t_cap;
  float scale_log2;
  void* o;
  int64_t o_sb, o_sh;
  int32_t out_bf16;
  float* lse;
  unsigned long long* trace;
};

struct Tiles {
  int32_t n_sink, loc_begin, n_tiles, pos;
};
__device__ __forceinline__ Tiles window_tiles(const PairParams& p, int bi) {
  int64_t L = p.seq_lens[bi];
  L = L < 1 ? 1 : (L > p.t_cap ? p.t_cap : L);
  Tiles t;
  t.pos = (int32_t)(L - 1);
  const int32_t last_tile = t.pos >> 7, tpb = p.b >> 7, QB = t.pos / p.b;
  int32_t sink_end = (QB + 1 < p.s ? QB + 1 : p.s) * tpb;
  if (sink_end > last_tile + 1) sink_end = last_tile + 1;
  int32_t lb = QB - p.l + 1;
  if (lb < p.s) lb = p.s;
  lb *= tpb;
  int32_t le = (QB + 1) * tpb;
  if (le > last_tile + 1) le = last_tile + 1;
  t.n_sink = sink_end;
  t.loc_begin = lb;
  t.n_tiles = sink_end + (le > lb ? le - lb : 0);
  return t;
}
__device__ __forceinline__ int32_t key0(const Tiles& t, int i) {
  return (i < t.n_sink ? i : t.loc_begin + (i - t.n_sink)) * 128;
}

// smem descriptor with SWIZZLE_64B (layout type 4): P is [key][32 heads] bf16, 64-byte rows
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                               uint32_t bar, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6, %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_commit_1sm_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}

#define PTRACE(slot, idx)                                                                                 \
  do {                                                                                                    \
    if (p.trace && blockIdx.x == 0 && (idx) < 16 && (threadIdx.x & 31) == 0) p.trace[(slot)*16 + (idx)] = clock64(); \
  } while (0)

__device__ __forceinline__ float m_used_at(const float (&m)[kHC], uint32_t lane) {
  float r = m[0];
#pragma unroll
  for (int j = 1; j < kHC; ++j) r = (j == (int)lane) ? m[j] : r;
  return r;
}

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    decode_pair_kernel(const __grid_constant__ PairParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int bi = (int)(blockIdx.x >> 1);
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  PTRACE(0, 0);
  const Tiles T = window_tiles(p, bi);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar(kBarFull + i), 1);
      mbar_init(bar(kBarEmpty + i), 2);  // both CTAs' UMMAs must have consumed the slot
    }
    mbar_init(bar(kBarQFull), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), kSmWarps);
      mbar_init(bar(kBarPFull + i), kSmWarps);
      mbar_init(bar(kBarOFull + i), 1);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(&p.v_map);
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_ptr_smem), kTmemCols);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;
  const int n = T.n_tiles;
  PTRACE(0, 1);

  if (warp == 0) {
    // ---------------- producer: Q (own heads), K / V stages (own half, multicast to the pair)
    const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
    if (elect_one()) {
      mbar_arrive_expect_tx(bar(kBarQFull), kQBytes);
      for (int c = 0; c < kChunks; ++c)
        tma_load_3d(sbase + kOffQ + c * (kHC * 128), &p.q_map, c * 64, kHC * (int)rank, bi, bar(kBarQFull), pol_q);
    }
    __syncwarp();
    uint32_t stage = 0, phase = 0;
    auto acquire = [&]() -> uint32_t {
      mbar_wait(bar(kBarEmpty + stage), phase ^ 1);
      return sbase + kOffRing + stage * kStageBytes;
    };
    auto next = [&]() {
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    };
    auto load_k = [&](int32_t k0) {
      for (int c = 0; c < kChunks; ++c) {
        const uint32_t dst = acquire();
        if (elect_one()) {
          mbar_arrive_expect_tx(bar(kBarFull + stage), kStageBytes);
          tma_load_3d_mc(dst + rank * 8192, &p.k_map, c * 64, k0 + 64 * (int)rank, bi, bar(kBarFull + stage), 3,
                         pol_kv);
        }
        __syncwarp();
        next();
      }
    };
    auto load_v = [&](int32_t k0) {
      for (int kq = 0; kq < 4; ++kq)
        for (int nh = 0; nh < 2; ++nh) {
          const uint32_t dst = acquire();
          if (elect_one()) {
            mbar_arrive_expect_tx(bar(kBarFull + stage), kStageBytes);
            for (int e = 2 * (int)rank; e < 2 * (int)rank + 2; ++e)
              tma_load_3d_mc(dst + e * 4096, &p.v_map, 256 * nh + 64 * e, k0 + 32 * kq, bi, bar(kBarFull + stage), 3,
                             pol_kv);
          }
          __syncwarp();
          next();
        }
    };
    load_k(key0(T, 0));
    for (int i = 1; i < n; ++i) {
      load_k(key0(T, i));
      load_v(key0(T, i - 1));
    }
    load_v(key0(T, n - 1));
  } else if (warp == 1) {
    // ---------------- UMMA issuer (each CTA issues its own cta_group::1 UMMAs)
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, kHC, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(128, kHC, true, true);
    const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
    const uint64_t dk = sdesc_sw128(sbase + kOffRing, 16, 1024);
    const uint64_t dv = sdesc_sw128(sbase + kOffRing, 4096, 1024);
    const uint64_t dp = sdesc_sw64(sbase + kOffP, 4096, 512);
    uint32_t stage = 0, phase = 0;
    auto next = [&]() {
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    };
    mbar_wait(bar(kBarQFull), 0);
    PTRACE(0, 2);
    auto issue_s = [&](uint32_t gi) {
      const uint32_t buf = gi & 1;
      mbar_wait(bar(kBarSFree + buf), ((gi >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int c = 0; c < kChunks; ++c) {
        mbar_wait(bar(kBarFull + stage), phase);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_1sm(tmem + kTmemS + 32 * buf, dk + (uint64_t)((kStageBytes * stage + 32 * k) >> 4),
                          dq + (uint64_t)((kHC * 128 * c + 32 * k) >> 4), idesc_s, (c | k) != 0);
          umma_commit_1sm_mc(bar(kBarEmpty + stage), 3);
        }
        __syncwarp();
        next();
      }
      if (elect_one()) umma_commit_1sm(bar(kBarSFull + buf));
      __syncwarp();
      PTRACE(1, gi);
    };
    auto issue_pv = [&](uint32_t gi) {
      const uint32_t buf = gi & 1;
      mbar_wait(bar(kBarPFull + buf), (gi >> 1) & 1);
      tc_fence_after();
      for (int kq = 0; kq < 4; ++kq)
        for (int nh = 0; nh < 2; ++nh) {
          mbar_wait(bar(kBarFull + stage), phase);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
              for (int dg = 0; dg < 2; ++dg)
                umma_bf16_1sm(tmem + kHC * (2 * nh + dg),
                              dv + (uint64_t)((kStageBytes * stage + 8192 * dg + 2048 * kk) >> 4),
                              dp + (uint64_t)((buf * kPBytes + (32 * kq + 16 * kk) * (kHC * 2)) >> 4), idesc_pv,
                              !(gi == 0 && kq == 0 && kk == 0));
            umma_commit_1sm_mc(bar(kBarEmpty + stage), 3);
          }
          __syncwarp();
          next();
        }
      if (elect_one()) umma_commit_1sm(bar(kBarOFull + buf));
      __syncwarp();
      PTRACE(2, gi);
    };
    for (int i = 0; i < n; ++i) {
      issue_s(i);
      if (i >= 1) issue_pv(i - 1);
    }
    issue_pv(n - 1);
  } else {
    // ---------------- softmax + epilogue (warps 2-5): TMEM lane = key of the tile, 32 heads per thread
    const uint32_t wq = warp & 3;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const float sl2 = p.scale_log2;
    float m_used[kHC], lpart[kHC];
#pragma unroll
    for (int j = 0; j < kHC; ++j) {
      m_used[j] = -INFINITY;
      lpart[j] = 0.f;
    }
    for (int i = 0; i < n; ++i) {
      const uint32_t buf = i & 1;
      const bool kvalid = key0(T, i) + 32 * (int32_t)wq + (int32_t)lane <= T.pos;
      mbar_wait(bar(kBarSFull + buf), (i >> 1) & 1);
      if (warp == 2) PTRACE(3, i);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(taddr + kTmemS + 32 * buf, v);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarSFree + buf));
      float* rb = red + buf * 4 * kHC;
      float wmax_mine = -INFINITY;
#pragma unroll
      for (int j = 0; j < kHC; ++j) {
        const float x = kvalid ? __uint_as_float(v[j]) : -INFINITY;
        float rr;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(rr) : "f"(x));
        if (j == (int)lane) wmax_mine = rr;
      }
      rb[wq * kHC + lane] = wmax_mine;
      named_bar_sync(1, 32 * kSmWarps);
      const float hmax = fmaxf(fmaxf(rb[lane], rb[kHC + lane]), fmaxf(rb[2 * kHC + lane], rb[3 * kHC + lane])) * sl2;
      float corr[kHC];
      bool any_resc = false;
#pragma unroll
      for (int j = 0; j < kHC; ++j) {
        const float tm = __shfl_sync(0xffffffffu, hmax, j);
        const bool resc = tm > m_used[j] + 8.0f;
        const float m_new = resc ? tm : m_used[j];
        corr[j] = resc ? ex2(m_used[j] - m_new) : 1.0f;
        any_resc |= resc;
        m_used[j] = m_new;
      }
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < kHC; j += 2) {
        const float e0 = kvalid ? ex2(fmaf(__uint_as_float(v[j]), sl2, -m_used[j])) : 0.f;
        const float e1 = kvalid ? ex2(fmaf(__uint_as_float(v[j + 1]), sl2, -m_used[j + 1])) : 0.f;
        lpart[j] = fmaf(lpart[j], corr[j], e0);
        lpart[j + 1] = fmaf(lpart[j + 1], corr[j + 1], e1);
        pk[j >> 1] = pack_bf16x2(e0, e1);
      }
      // P row = key (64 B = 32 heads), SWIZZLE_64B: 16-byte unit u stored at u ^ ((row >> 1) & 3)
      const uint32_t krow = 32 * wq + lane;
      const uint32_t prow = sbase + kOffP + buf * kPBytes + krow * 64;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        st_shared_v4(prow + ((u ^ ((krow >> 1) & 3)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      if (i > 0) {
        mbar_wait(bar(kBarOFull + ((i - 1) & 1)), ((i - 1) >> 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, any_resc)) {
#pragma unroll 1
          for (int gg = 0; gg < 4; ++gg) {
            uint32_t ov[32];
            tmem_ld32(taddr + kHC * gg, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr[j]);
            tmem_st32(taddr + kHC * gg, ov);
          }
          tmem_wait_st();
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarPFull + buf));
      if (warp == 2) PTRACE(4, i);
    }
    // ---------------- epilogue: l per head, O^T / l -> bf16 [head][dim] in smem -> 16-byte stores
    mbar_wait(bar(kBarOFull + ((n - 1) & 1)), ((n - 1) >> 1) & 1);
    if (warp == 2) PTRACE(5, 0);
    tc_fence_after();
    float lmine = 0.f;
#pragma unroll
    for (int j = 0; j < kHC; ++j) {
      float x = lpart[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (j == (int)lane) lmine = x;
    }
    float* ls = red + (n & 1) * 4 * kHC;  // the exchange buffer the last tile did not use
    ls[wq * kHC + lane] = lmine;
    named_bar_sync(1, 32 * kSmWarps);
    const float lh = (ls[lane] + ls[kHC + lane]) + (ls[2 * kHC + lane] + ls[3 * kHC + lane]);
    float inv[kHC];
#pragma unroll
    for (int j = 0; j < kHC; ++j) inv[j] = 1.0f / __shfl_sync(0xffffffffu, lh, j);
    // staging: the ring is idle (every stage of both CTAs consumed); [32 heads][512 dims] bf16 / fp32
    const int esz = p.out_bf16 ? 2 : 4;
    uint8_t* stg = smem + kOffRing;
#pragma unroll 1
    for (int gg = 0; gg < 4; ++gg) {
      uint32_t ov[32];
      tmem_ld32(taddr + kHC * gg, ov);
      tmem_wait_ld();
      const int dim = 128 * gg + 32 * (int)wq + (int)lane;
#pragma unroll
      for (int j = 0; j < kHC; ++j) {
        const float val = __uint_as_float(ov[j]) * inv[j];
        if (p.out_bf16)
          *reinterpret_cast<unsigned short*>(stg + (j * kDv + dim) * 2) = (unsigned short)(pack_bf16x2(val, 0.f) & 0xFFFFu);
        else
          *reinterpret_cast<float*>(stg + (j * kDv + dim) * 4) = val;
      }
    }
    if (p.lse && wq == 0)
      p.lse[(int64_t)bi * kH + kHC * rank + lane] = (m_used_at(m_used, lane) + __log2f(lh)) * 0.69314718055994531f;
    named_bar_sync(1, 32 * kSmWarps);
    const int tid = (int)threadIdx.x - 64;  // 0..127
    const int row_bytes = kDv * esz, chunks = kHC * row_bytes / 16;
    for (int k = tid; k < chunks; k += 32 * kSmWarps) {
      const int j = (k * 16) / row_bytes, off = (k * 16) % row_bytes;
      const uint4 w = *reinterpret_cast<const uint4*>(stg + j * row_bytes + off);
      char* dst = reinterpret_cast<char*>(p.o) + ((int64_t)bi * p.o_sb + (int64_t)(kHC * rank + j) * p.o_sh) * esz + off;
      st_global_v4(dst, w.x, w.y, w.z, w.w);
    }
  }
  if (warp == 2) PTRACE(5, 1);
  __syncwarp();
  tc_fence_before();
  cluster_sync();  // the partner may still multicast into this CTA until both are done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, kTmemCols);
  }
}

}  // namespace

bool decode_pair_eligible(const AttnProblem& a, int sms) {
  return a.sparse && a.heads == kH && a.b % 128 == 0 && 2 * (int64_t)a.batch <= sms && a.n_kv < (1ll << 31);
}

unsigned long long* g_pair_trace = nullptr;

cudaError_t launch_decode_pair(const AttnProblem& a, cudaStream_t st) {
  PairParams p;
  memset(&p, 0, sizeof(p));
  p.seq_lens = a.seq_lens;
  p.batch = a.batch;
  p.s = a.s;
  p.l = a.l;
  p.b = a.b;
  p.t_cap = a.n_kv;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.o = a.o;
  p.o_sb = a.o_sb;
  p.o_sh = a.o_sh;
  p.out_bf16 = a.out_bf16;
  p.lse = a.lse;
  p.trace = g_pair_trace;
  const KvSeg& s = a.kv.seg[0];
  if (!encode_3d(&p.q_map, a.q, kDqk, kH, a.batch, a.q_sh, a.q_sb, kHC)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.k_map, s.k, kDqk, (uint64_t)a.n_kv, a.batch, s.k_st, s.k_sb, 64)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.v_map, s.v, kDv, (uint64_t)a.n_kv, a.batch, s.v_st, s.v_sb, 32)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(decode_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  decode_pair_kernel<<<2 * a.batch, kThreads, kSmemAlloc, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza

extern "C" void loza_debug_set_pair_trace(void* dev_ptr) { loza::g_pair_trace = (unsigned long long*)dev_ptr; }
