// SSA decode with a CTA pair per sequence (Eq. 4 at p = seq_len - 1).
//
// Design:
//  * Cluster of 2 per sequence; CTA r streams half of the sequence's selected 128-key tiles, so each SM
//    receives half of the window and 2B SMs pull from HBM together.
//  * Transposed products keep M = 128 (full-rate UMMA; M = 64, heads as rows, runs at half rate):
//    S^T[key][head] = K Q^T (A = K chunk 128 keys x 64 dims, B = Q chunk, N = 64 heads) and
//    O^T[dim][head] += V^T P (A = V slab MN-major, B = P [key][head] MN-major, N = 64 heads).
//    TMEM: O^T 4 groups x 64 cols (lanes = 128 dims of a group), S^T 2 buffers x 64 cols at 256.
//  * Per CTA: warp 0 TMA producer (Q: 9 per-chunk barriers, issued first; ring of 7 x 16 KB: K chunk
//    128 keys x 64 dims, V slab 32 keys x 256 dims), warp 1 UMMA issuer (warp-uniform, elected lane),
//    warps 2-9 softmax (per-head max over keys with redux.sync, then over the 4 key-quarter warps).
//  * Merge (the two halves of the window): CTA r finalises dims [256 r, 256 r + 256) for all 64 heads.
//    Each CTA stages the partner's dims of its unnormalised O^T (fp32) and its per-head (m, l) in its idle
//    Q region and sends them with ONE bulk DSMEM copy (cp.async.bulk shared::cluster; ~18 B/clk/SM measured,
//    tools/dsmem_bw.cu, vs ~15 for st.shared::cluster and ~11 through L2); all 8 softmax warps combine,
//    stage bf16 [64 heads x 64 dims] swizzled boxes and TMA-store them.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {
using namespace sm100;

constexpr int kDqk = 576, kDv = 512, kChunks = 9, kH = 64;
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 softmax / merge
constexpr int kStageBytes = 32768;  // ring item: 2 K chunks (128 keys x 128 dims) or 2 V slabs (64 keys x 256 dims)
constexpr int kStages = 3;
constexpr int kHalf = 16384;
constexpr int kQBytes = kChunks * 64 * 128;  // 73728
constexpr int kPBytes = 2 * 64 * 128;        // 16384 per buffer: P [128 keys][64 heads] bf16
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffRing = kOffP + 2 * kPBytes;
constexpr int kOffBar = kOffRing + kStages * kStageBytes;  // 221184
constexpr int kBarRingFull = 0;
constexpr int kBarRingEmpty = kBarRingFull + kStages;
constexpr int kBarQFull = kBarRingEmpty + kStages;  // [9]
constexpr int kBarSFull = kBarQFull + kChunks;       // [2]
constexpr int kBarSFree = kBarSFull + 2;             // [2]
constexpr int kBarPFull = kBarSFree + 2;             // [2]
constexpr int kBarOFull = kBarPFull + 2;             // [2]
constexpr int kBarRecv = kBarOFull + 2;              // partner's half landed
constexpr int kNumBars = kBarRecv + 1;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffRed = (kOffTmemPtr + 4 + 15) & ~15;  // float [2 buf][4 key quarters][64 heads]
constexpr int kOffML = kOffRed + 2 * 4 * 64 * 4;       // float mloc[64], lloc[64]
constexpr int kOffW = kOffML + 2 * 64 * 4;             // float merge weights w_own[64], w_par[64]
constexpr int kSmemUsed = kOffW + 2 * 64 * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");
// merge buffers (all idle once both CTAs finished their tiles)
constexpr int kSendO = 2 * 128 * 2 * 128;        // [2 groups][128 dims][2 head halves][32 heads] fp32 = 64 KB
constexpr int kSendBytes = kSendO + 2 * 64 * 4;  // + m[64], l[64]
constexpr int kOffSend = kOffQ;                  // own Q region
constexpr int kOffRecv = kOffRing;               // partner writes into this CTA's ring
constexpr int kOffOut = kOffP;                   // bf16 [4 boxes][64 heads][64 dims] in the idle P buffers
static_assert(kSendBytes <= kQBytes, "send staging fits the Q region");
static_assert(kSendBytes <= kStages * kStageBytes, "receive staging fits the ring");
static_assert(4 * 8192 <= 2 * kPBytes, "output staging fits the P buffers");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemS = 256;  // S^T buffer b: 128 lanes (keys) x 64 cols (heads) at 256 + 64 b
constexpr uint32_t kSoftmaxWarps = 8;
constexpr uint32_t kSmThreads = 32 * kSoftmaxWarps;

struct PairParams {
  CUtensorMap q_map, k_map, v_map, o_map;
  const int32_t* seq_lens;
  int32_t batch, s, l, b;
  int32_t ring;  // k/v is the bounded ring cache (ring_cache.cu): tile rows are remapped, positions are not
  int64_t t_cap;
  float scale_log2;
  void* o;
  int64_t o_sb, o_sh;
  int32_t out_bf16;
  float* lse;
  unsigned long long* trace;  // debug timeline of CTA 0 (NULL in production)
};

struct SeqTiles {
  int32_t n_sink, loc_begin, n_tiles;
  int32_t pos;  // query position p = seq_len - 1 (< 2^31)
};

// the selected 128-key tiles of the query at p = seq_len - 1 (closed form of select_blocks.cu)
__device__ __forceinline__ SeqTiles seq_tiles(const PairParams& p, int bi) {
  int64_t L = p.seq_lens[bi];
  L = L < 1 ? 1 : (L > p.t_cap ? p.t_cap : L);
  SeqTiles t;
  t.pos = (int32_t)(L - 1);
  const int32_t last_tile = t.pos >> 7;
  const int32_t tpb = p.b >> 7, QB = t.pos / p.b;
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
__device__ __forceinline__ int32_t tile_k0(const SeqTiles& t, int i) {
  return (i < t.n_sink ? i : t.loc_begin + (i - t.n_sink)) * 128;
}
// cache row of the 128-key tile at absolute key k0: identity, or the ring slot of its block
__device__ __forceinline__ int32_t kv_row(const PairParams& p, int32_t k0) {
  if (!p.ring) return k0;
  const int32_t kb = k0 / p.b;
  if (kb < p.s) return k0;
  return p.s * p.b + ((kb - p.s) % p.l) * p.b + (k0 - kb * p.b);
}

#define DTRACE(slot, idx)                                                                        \
  do {                                                                                           \
    if (p.trace && blockIdx.x == 0 && (idx) < 32 && (threadIdx.x & 31) == 0) p.trace[(slot)*32 + (idx)] = clock64(); \
  } while (0)

// m[lane] from a per-thread register array indexed by the lane id (unrolled select, keeps m in registers)
__device__ __forceinline__ float m_used_lane(const float (&m)[32], uint32_t lane) {
  float r = m[0];
#pragma unroll
  for (int j = 1; j < 32; ++j) r = (j == (int)lane) ? m[j] : r;
  return r;
}

__device__ __forceinline__ void bulk_copy_to_cluster(uint32_t dst_cluster, uint32_t src, uint32_t bytes,
                                                     uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
      "r"(src), "r"(bytes), "r"(bar_cluster)
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    decode_pair_kernel(const __grid_constant__ PairParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  float* mloc = reinterpret_cast<float*>(smem + kOffML);
  float* lloc = mloc + 64;
  const uint32_t rank = cluster_ctarank(), partner = rank ^ 1;
  const int bi = (int)(blockIdx.x >> 1);

  DTRACE(0, 0);
  if (p.trace && threadIdx.x == 0) {  // per-CTA wall-clock span (globaltimer, ns) after the CTA-0 timeline
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[12 * 32 + 2 * blockIdx.x] = g;
  }
  // Programmatic dependent launch: let the next kernel in the stream be scheduled now (its CTAs wait in
  // griddepcontrol.wait until this grid has completed), and do the input-independent setup before waiting
  // for the previous one. Every read of q, the cache or seq_lens comes after the wait.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar(kBarRingFull + i), 1);
      mbar_init(bar(kBarRingEmpty + i), 1);
    }
    for (int i = 0; i < kChunks; ++i) mbar_init(bar(kBarQFull + i), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), kSoftmaxWarps);
      mbar_init(bar(kBarPFull + i), kSoftmaxWarps);
      mbar_init(bar(kBarOFull + i), 1);
    }
    mbar_init(bar(kBarRecv), 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar(kBarRecv), kSendBytes);  // armed now; the partner's bulk copy completes it
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(&p.v_map);
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    mloc[i] = -INFINITY;
    lloc[i] = 0.f;
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_ptr_smem), kTmemCols);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const SeqTiles st = seq_tiles(p, bi);
  const int mid = (st.n_tiles + 1) / 2;
  const int t0 = rank ? mid : 0, t1 = rank ? st.n_tiles : mid;  // rank 1 may get none
  const int n = t1 - t0;
  const bool has_tiles = n > 0;
  if (threadIdx.x == 0 && has_tiles) {  // Q first: the first S waits on it chunk by chunk
    const uint64_t pol_q = policy_evict_first();
    for (int c = 0; c < kChunks; ++c) {
      mbar_arrive_expect_tx(bar(kBarQFull + c), 8192);
      tma_load_3d(sbase + kOffQ + c * 8192, &p.q_map, c * 64, 0, bi, bar(kBarQFull + c), pol_q);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;
  DTRACE(0, 1);

  if (warp == 0 && has_tiles) {
    // ----------------------------------------------------- TMA producer (warp-uniform, elected lane issues)
    const uint64_t pol_kv = policy_evict_last();
    uint32_t stage = 0, phase = 0;
    auto acquire = [&]() -> uint32_t {
      mbar_wait(bar(kBarRingEmpty + stage), phase ^ 1);
      return sbase + kOffRing + stage * kStageBytes;
    };
    auto next = [&]() {
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    };
    // 32 KB items (half the per-item wait/commit overhead of 16 KB items): K chunks {2j, 2j + 1} (chunk 8
    // alone), V slabs of keys 64 kp .. 64 kp + 63 (two 32-key boxes) x dim chunks 4 nh .. 4 nh + 3
    auto load_k = [&](int32_t k0) {
      for (int j = 0; j < (kChunks + 1) / 2; ++j) {
        const uint32_t dst = acquire();
        const int nc = 2 * j + 1 < kChunks ? 2 : 1;
        if (elect_one()) {
          mbar_arrive_expect_tx(bar(kBarRingFull + stage), nc * kHalf);
          for (int sub = 0; sub < nc; ++sub)
            tma_load_3d(dst + kHalf * sub, &p.k_map, (2 * j + sub) * 64, k0, bi, bar(kBarRingFull + stage), pol_kv);
        }
        __syncwarp();
        next();
      }
    };
    auto load_v = [&](int32_t k0) {
      for (int kp = 0; kp < 2; ++kp)
        for (int nh = 0; nh < 2; ++nh) {
          const uint32_t dst = acquire();
          if (elect_one()) {
            mbar_arrive_expect_tx(bar(kBarRingFull + stage), kStageBytes);
            // 4-D boxes: 32 keys x dim chunks 4 nh .. 4 nh + 3 (smem [chunk][32 keys][64 dims]) per half
            for (int sub = 0; sub < 2; ++sub)
              tma_load_4d(dst + kHalf * sub, &p.v_map, 0, k0 + 32 * (2 * kp + sub), 4 * nh, bi,
                          bar(kBarRingFull + stage), pol_kv);
          }
          __syncwarp();
          next();
        }
    };
    load_k(kv_row(p, tile_k0(st, t0)));
    for (int i = t0 + 1; i < t1; ++i) {
      load_k(kv_row(p, tile_k0(st, i)));
      load_v(kv_row(p, tile_k0(st, i - 1)));
    }
    load_v(kv_row(p, tile_k0(st, t1 - 1)));
  } else if (warp == 1 && has_tiles) {
    // ----------------------------------------------------- UMMA issuer (warp-uniform, elected lane issues)
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 64, true, true);
    const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
    const uint64_t dr_k = sdesc_sw128(sbase + kOffRing, 16, 1024);
    const uint64_t dr_v = sdesc_sw128(sbase + kOffRing, 4096, 1024);
    const uint64_t dp = sdesc_sw128(sbase + kOffP, 8192, 1024);
    uint32_t stage = 0, phase = 0;
    auto next = [&]() {
      if (++stage == kStages) {
        stage = 0;
        phase ^= 1;
      }
    };
    auto issue_s = [&](uint32_t gi) {
      const uint32_t buf = gi & 1;
      DTRACE(1, gi);
      mbar_wait(bar(kBarSFree + buf), ((gi >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + kTmemS + 64 * buf;
      long long kw = 0;
      for (int j = 0; j < (kChunks + 1) / 2; ++j) {
        const int nc = 2 * j + 1 < kChunks ? 2 : 1;
        const long long w0 = clock64();
        if (gi == 0)
          for (int sub = 0; sub < nc; ++sub) mbar_wait(bar(kBarQFull + 2 * j + sub), 0);
        mbar_wait(bar(kBarRingFull + stage), phase);
        kw += clock64() - w0;
        tc_fence_after();
        if (elect_one()) {
          for (int sub = 0; sub < nc; ++sub) {
            const int cc = 2 * j + sub;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16_1sm(d, dr_k + (uint64_t)((kStageBytes * stage + kHalf * sub + 32 * k) >> 4),
                            dq + (uint64_t)((8192 * cc + 32 * k) >> 4), idesc_s, (cc | k) != 0);
          }
          umma_commit_1sm(bar(kBarRingEmpty + stage));
        }
        __syncwarp();
        next();
      }
      if (elect_one()) umma_commit_1sm(bar(kBarSFull + buf));
      __syncwarp();
      DTRACE(2, gi);
      if (p.trace && blockIdx.x == 0 && gi < 32 && lane == 0) p.trace[12 * 32 + 4 * p.batch + gi] = kw;
    };
    auto issue_pv = [&](uint32_t gi, bool first) {
      const uint32_t buf = gi & 1;
      DTRACE(3, gi);
      mbar_wait(bar(kBarPFull + buf), (gi >> 1) & 1);
      DTRACE(4, gi);
      tc_fence_after();
      long long vw = 0;
      for (int kp = 0; kp < 2; ++kp)
        for (int nh = 0; nh < 2; ++nh) {
          const long long w0 = clock64();
          mbar_wait(bar(kBarRingFull + stage), phase);
          vw += clock64() - w0;
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int sub = 0; sub < 2; ++sub) {
              const int kq = 2 * kp + sub;
#pragma unroll
              for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int dg = 0; dg < 2; ++dg)
                  umma_bf16_1sm(tmem + 64 * (2 * nh + dg),
                                dr_v + (uint64_t)((kStageBytes * stage + kHalf * sub + 8192 * dg + 2048 * kk) >> 4),
                                dp + (uint64_t)((buf * kPBytes + (32 * kq + 16 * kk) * 128) >> 4), idesc_pv,
                                !(first && kq == 0 && kk == 0));
            }
            umma_commit_1sm(bar(kBarRingEmpty + stage));
          }
          __syncwarp();
          next();
        }
      if (elect_one()) umma_commit_1sm(bar(kBarOFull + buf));
      __syncwarp();
      DTRACE(5, gi);
      if (p.trace && blockIdx.x == 0 && gi < 32 && lane == 0) p.trace[12 * 32 + 4 * p.batch + 32 + gi] = vw;
    };
    for (int i = 0; i < n; ++i) {
      issue_s((uint32_t)i);
      if (i >= 1) issue_pv((uint32_t)(i - 1), i - 1 == 0);
    }
    issue_pv((uint32_t)(n - 1), n == 1);
  } else if (warp >= 2 && has_tiles) {
    // ----------------------------------------------------- softmax (warps 2..9)
    // TMEM lane quarter wq = warp % 4: S^T lanes = keys 32 wq .. 32 wq + 31 of the tile. Column half
    // ch = (warp - 2) / 4 selects heads [32 ch, 32 ch + 32): a thread holds one key's 32 heads. Per-head maxima
    // over keys: redux.sync.max.f32 within the warp, then the 4 key-quarter warps through shared memory.
    const uint32_t wq = warp & 3;
    const uint32_t ch = (warp - 2) >> 2;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const float sl2 = p.scale_log2;
    float m_used[32], lpart[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      m_used[j] = -INFINITY;
      lpart[j] = 0.f;
    }
    for (int i = 0; i < n; ++i) {
      const uint32_t gi = (uint32_t)i, buf = gi & 1;
      const int32_t key = tile_k0(st, t0 + i) + 32 * (int32_t)wq + (int32_t)lane;
      const bool kvalid = key <= st.pos;
      if (warp == 2) DTRACE(6, gi);
      mbar_wait(bar(kBarSFull + buf), (gi >> 1) & 1);
      if (warp == 2) DTRACE(7, gi);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(taddr + kTmemS + 64 * buf + 32 * ch, v);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarSFree + buf));
      float* rb = red + buf * 256;
      float wmax_mine = -INFINITY;  // lane j keeps head 32 ch + j
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = kvalid ? __uint_as_float(v[j]) : -INFINITY;
        float r;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
        if (j == (int)lane) wmax_mine = r;
      }
      rb[wq * 64 + 32 * ch + lane] = wmax_mine;
      named_bar_sync(1, kSmThreads);
      const float hmax = fmaxf(fmaxf(rb[32 * ch + lane], rb[64 + 32 * ch + lane]),
                               fmaxf(rb[128 + 32 * ch + lane], rb[192 + 32 * ch + lane])) * sl2;
      uint32_t pk[16];
      bool any_resc = false;
      float corr[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float tm = __shfl_sync(0xffffffffu, hmax, j);
        const bool resc = tm > m_used[j] + 8.0f;
        const float m_new = resc ? tm : m_used[j];
        corr[j] = resc ? ex2(m_used[j] - m_new) : 1.0f;
        any_resc |= resc;
        m_used[j] = m_new;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float e0 = kvalid ? ex2(fmaf(__uint_as_float(v[j]), sl2, -m_used[j])) : 0.f;
        const float e1 = kvalid ? ex2(fmaf(__uint_as_float(v[j + 1]), sl2, -m_used[j + 1])) : 0.f;
        lpart[j] = fmaf(lpart[j], corr[j], e0);
        lpart[j + 1] = fmaf(lpart[j + 1], corr[j + 1], e1);
        pk[j >> 1] = pack_bf16x2(e0, e1);
      }
      // P[key][head] row (128 B = 64 heads), this thread's 64 B at units 4 ch .. 4 ch + 3
      const uint32_t krow = 32 * wq + lane;
      const uint32_t prow = sbase + kOffP + buf * kPBytes + krow * 128;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        st_shared_v4(prow + (((4 * ch + u) ^ (krow & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2],
                     pk[4 * u + 3]);
      if (i > 0) {
        const uint32_t gp = gi - 1;
        mbar_wait(bar(kBarOFull + (gp & 1)), (gp >> 1) & 1);
        tc_fence_after();
        // corr is per head: identical in every thread with this ch, so the warp decision is uniform
        if (__any_sync(0xffffffffu, any_resc)) {
#pragma unroll 1
          for (int gg = 0; gg < 4; ++gg) {  // O^T columns of this warp's heads in each 128-dim group
            uint32_t ov[32];
            tmem_ld32(taddr + 64 * gg + 32 * ch, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr[j]);
            tmem_st32(taddr + 64 * gg + 32 * ch, ov);
          }
          tmem_wait_st();
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarPFull + buf));
      if (warp == 2) DTRACE(8, gi);
    }
    // l[h] = sum over the 128 key lanes of lpart[h]; O^T is final once the last PV completed
    const uint32_t gl = (uint32_t)(n - 1);
    mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
    tc_fence_after();
    float lmine = 0.f;  // lane j: this warp's key-quarter sum for head 32 ch + j
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float x = lpart[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (j == (int)lane) lmine = x;
    }
    float* ls = red + ((gl + 1) & 1) * 256;
    ls[wq * 64 + 32 * ch + lane] = lmine;
    named_bar_sync(1, kSmThreads);
    if (wq == 0) {
      mloc[32 * ch + lane] = m_used_lane(m_used, lane);
      lloc[32 * ch + lane] =
          (ls[32 * ch + lane] + ls[64 + 32 * ch + lane]) + (ls[128 + 32 * ch + lane] + ls[192 + 32 * ch + lane]);
    }
  }
  __syncwarp();
  if (warp == 2) DTRACE(9, 0);

  // ---------------------------------------------------------------- merge of the two halves
  const uint32_t wq = warp & 3, ch = (warp - 2) >> 2;
  const uint32_t taddr = tmem + ((wq * 32) << 16);
  const uint32_t t = wq * 32 + lane;  // TMEM lane = dim within a 128-dim group
  if (warp >= 2) {
    named_bar_sync(1, kSmThreads);  // mloc / lloc written
    // stage the partner's dims (groups 2 partner + gk) of O^T: [gk][t][ch][32 heads] fp32, 16-B units swizzled
#pragma unroll 1
    for (int gk = 0; gk < 2; ++gk) {
      uint32_t ov[32];
      tmem_ld32(taddr + 64 * (2 * partner + gk) + 32 * ch, ov);  // (undefined without tiles: masked)
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) ov[j] = has_tiles ? ov[j] : 0u;
      const uint32_t row = sbase + kOffSend + ((gk * 128 + t) * 2 + ch) * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q) st_shared_v4(row + ((q ^ (t & 7)) << 4), ov[4 * q], ov[4 * q + 1], ov[4 * q + 2], ov[4 * q + 3]);
    }
    if (wq == 0) {
      float* sml = reinterpret_cast<float*>(smem + kOffSend + kSendO);
      sml[32 * ch + lane] = mloc[32 * ch + lane];
      sml[64 + 32 * ch + lane] = lloc[32 * ch + lane];
    }
    fence_proxy_async_smem();
  }
  tc_fence_before();
  cluster_sync();  // #1: both CTAs finished their tiles (rings idle) and staged their halves
  tc_fence_after();
  if (threadIdx.x == 64)
    bulk_copy_to_cluster(mapa(sbase + kOffRecv, partner), sbase + kOffSend, kSendBytes, mapa(bar(kBarRecv), partner));
  if (warp >= 2) {
    mbar_wait(bar(kBarRecv), 0);
    if (warp == 2) DTRACE(10, 0);
    const float* rml = reinterpret_cast<const float*>(smem + kOffRecv + kSendO);
    float* wsm = reinterpret_cast<float*>(smem + kOffW);
    const int tid = (int)threadIdx.x - 64;
    if (tid < 64) {  // per-head weights: O = (w_own O_own + w_par O_par), (m, l) of both halves
      const int h = tid;
      const float mo = mloc[h], lo_ = lloc[h], mp = rml[h], lp = rml[64 + h];
      const float mt = fmaxf(mo, mp);
      const float wo = lo_ > 0.f ? ex2(mo - mt) : 0.f, wp = lp > 0.f ? ex2(mp - mt) : 0.f;
      const float lt = wo * lo_ + wp * lp, inv = 1.0f / lt;
      wsm[h] = wo * inv;
      wsm[64 + h] = wp * inv;
      if (p.lse && (h >> 5) == (int)rank) p.lse[(int64_t)bi * kH + h] = (mt + __log2f(lt)) * 0.69314718055994531f;
    }
    named_bar_sync(1, kSmThreads);
    const uint8_t* rb = smem + kOffRecv;
#pragma unroll 1
    for (int gk = 0; gk < 2; ++gk) {
      uint32_t own[32];
      tmem_ld32(taddr + 64 * (2 * rank + gk) + 32 * ch, own);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) own[j] = has_tiles ? own[j] : 0u;
      const uint8_t* row = rb + ((gk * 128 + t) * 2 + ch) * 128;
      const int dl = 128 * gk + (int)t;  // dim within this CTA's 256
      const uint32_t box = sbase + kOffOut + (dl >> 6) * 8192, col = (uint32_t)(dl & 63);
      float* ob = reinterpret_cast<float*>(p.o) + (int64_t)bi * p.o_sb + 256 * rank + dl;  // fp32 output only
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = *reinterpret_cast<const float4*>(row + ((q ^ (t & 7)) << 4));
        const float4 wo4 = *reinterpret_cast<const float4*>(wsm + 32 * ch + 4 * q);  // broadcast reads
        const float4 wp4 = *reinterpret_cast<const float4*>(wsm + 64 + 32 * ch + 4 * q);
        const float pv[4] = {f.x, f.y, f.z, f.w}, wo[4] = {wo4.x, wo4.y, wo4.z, wo4.w},
                    wp[4] = {wp4.x, wp4.y, wp4.z, wp4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = 4 * q + e;
          const uint32_t h = 32 * ch + j;
          const float val = fmaf(__uint_as_float(own[j]), wo[e], pv[e] * wp[e]);
          if (p.out_bf16) {
            // [box = dl / 64][head][64 dims] bf16, 128-B rows, 16-B units swizzled by head & 7
            const uint32_t a = box + h * 128 + (((col >> 3) ^ (h & 7)) << 4) + (col & 7) * 2;
            asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)(pack_bf16x2(val, 0.f) & 0xFFFFu)));
          } else {
            ob[(int64_t)h * p.o_sh] = val;
          }
        }
      }
    }
    if (p.out_bf16) {
      fence_proxy_async_smem();
      named_bar_sync(1, kSmThreads);
      if (warp == 2 && lane == 0) {
        for (int m = 0; m < 4; ++m) tma_store_3d(&p.o_map, sbase + kOffOut + m * 8192, 256 * (int)rank + 64 * m, 0, bi);
        bulk_commit_group();
        bulk_wait_group_read0();  // staging read before shared memory is released; the stores drain on their own
      }
    }
  }
  if (warp == 2) DTRACE(11, 0);
  if (p.trace && threadIdx.x == 64) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[12 * 32 + 2 * blockIdx.x + 1] = g;
  }
  tc_fence_before();
  cluster_sync();  // #2: both bulk copies landed before either CTA's shared memory goes away
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, kTmemCols);
  }
}

}  // namespace

unsigned long long* g_pair_trace = nullptr;

cudaError_t launch_decode_pair(const AttnProblem& a, cudaStream_t st) {
  if (a.heads != kH) return cudaErrorNotSupported;
  if (a.n_kv >= (1ll << 31)) return cudaErrorNotSupported;
  PairParams p;
  memset(&p, 0, sizeof(p));
  p.seq_lens = a.seq_lens;
  p.batch = a.batch;
  p.s = a.s;
  p.l = a.l;
  p.b = a.b;
  p.ring = a.ring;
  p.t_cap = a.ring ? (int64_t)0x7FFFFFFF : a.n_kv;  // ring: positions are absolute, any length
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.o = a.o;
  p.o_sb = a.o_sb;
  p.o_sh = a.o_sh;
  p.out_bf16 = a.out_bf16;
  p.lse = a.lse;
  p.trace = g_pair_trace;
  const KvSeg& s = a.kv.seg[0];
  if (!encode_3d(&p.q_map, a.q, kDqk, kH, a.batch, a.q_sh, a.q_sb, 64)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.k_map, s.k, kDqk, (uint64_t)a.n_kv, a.batch, s.k_st, s.k_sb, 128)) return cudaErrorInvalidValue;
  if (!encode_4d_chunks(&p.v_map, s.v, kDv, (uint64_t)a.n_kv, a.batch, s.v_st, s.v_sb, 32, 4))
    return cudaErrorInvalidValue;
  if (a.out_bf16 && !encode_3d(&p.o_map, a.o, kDv, kH, a.batch, a.o_sh, a.o_sb, 64)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(decode_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * a.batch));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemAlloc;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, decode_pair_kernel, p);
  if (le != cudaSuccess) return le;
  count_launch();
  return cudaGetLastError();
}

// pair mode: the pair-cooperative kernel (attn_tc_decode_coop.cu) unless LOZA_DECODE_KERNEL=pair selects the
// key-split pair kernel above (kept for A/B measurement)
cudaError_t launch_decode_pair_any(const AttnProblem& a, cudaStream_t st) {
  static const int use_split = [] {
    const char* e = getenv("LOZA_DECODE_KERNEL");
    return e && strcmp(e, "pair") == 0 ? 1 : 0;
  }();
  return use_split ? launch_decode_pair(a, st) : launch_decode_coop(a, st);
}

// pair mode: SSA, 64 heads, whole-tile blocks, and 2 CTAs per sequence fit in one wave
bool decode_pair_eligible(const AttnProblem& a, int sms) {
  return a.sparse && a.heads == kH && a.b % 128 == 0 && 2 * (int64_t)a.batch <= sms && a.n_kv < (1ll << 31);
}

}  // namespace loza

extern "C" void loza_debug_set_pair_trace(void* dev_ptr) { loza::g_pair_trace = (unsigned long long*)dev_ptr; }
