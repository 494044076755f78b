// SSA decode with a CTA pair per sequence (Eq. 4 at p = seq_len - 1): cluster of 2,
// CTA r streams half of the sequence's window tiles (so each SM receives only half of the window:
// one SM's TMA receive rate caps at ~67 B/clk, tools/tma_bw.cu), then the two partial results are
// merged through distributed shared memory (no global partials): CTA r finalises heads [32r, 32r+32),
// its partner sends those heads' unnormalised O^T and (m, l) with st.shared::cluster, and the output is
// staged in shared memory for 16-byte coalesced stores. Compute uses transposed products (M = 128:
// S^T = K Q^T over keys x heads, O^T += V^T P over dims x heads). The flattened split-KV kernel
// (attn_tc_decode.cu) serves larger batches and the full-attention comparator.
//
// Design:
//  * The 64 heads of one token are the MMA rows (M = 64, cta_group::1): S = Q K^T
//    (N = 128 keys per tile, K = 576), P V with N = 256 per half of d_v. TMEM uses
//    the M=64 half-lane layout: O[:, 0:256) in lanes 0-15 of each sub-partition,
//    O[:, 256:512) in lanes 16-31 (same columns 0..255), S (double buffered) in lanes
//    0-15 at columns 256..511. A 32x32b TMEM access of columns 0..255 touches only O.
//  * Split-KV over a flattened tile space: every sequence b contributes T_b tiles of
//    128 keys (computed on the device from seq_lens, so a decode step is CUDA-graph
//    capturable); CTA c takes tiles [c*T/G, (c+1)*T/G). A (CTA, sequence) piece that
//    covers the whole sequence writes O directly; otherwise it writes a partial
//    (unnormalised O, running max, running sum) to ws slot c + b, and the last CTA to
//    finish a sequence (device counter, self-resetting) merges the pieces in CTA order
//    (deterministic). SSA decode reads (s+l)*b rows per sequence whatever the context.
//  * Per CTA: warp 0 TMA producer (16 KB stages: K chunk 128 keys x 64 dims, V slab
//    32 keys x 256 dims), warp 1 UMMA issuer (warp-uniform, elected lane issues),
//    warps 2-9 softmax / merge / epilogue (two warps per TMEM sub-partition, each takes
//    64 of a row's 128 logits). Tile lists are computed once per CTA, in parallel, into
//    shared memory (no per-role 64-bit divisions).
#include <math.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {
using namespace sm100;

constexpr int kDqk = 576, kDv = 512, kChunks = 9, kH = 64;
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 softmax
constexpr int kMaxBatch = 896;
constexpr int kStageBytes = 16384;
constexpr int kStages = 7;
constexpr int kQBytes = kChunks * 64 * 128;  // 73728
constexpr int kPBytes = 2 * 64 * 128;        // 16384 per buffer
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffRing = kOffP + 2 * kPBytes;
constexpr int kOffBar = kOffRing + kStages * kStageBytes;
constexpr int kBarRingFull = 0;
constexpr int kBarRingEmpty = kBarRingFull + kStages;
constexpr int kBarQFull = kBarRingEmpty + kStages;
constexpr int kBarQEmpty = kBarQFull + 1;
constexpr int kBarSFull = kBarQEmpty + 1;  // [2]
constexpr int kBarSFree = kBarSFull + 2;   // [2]
constexpr int kBarPFull = kBarSFree + 2;   // [2]
constexpr int kBarOFull = kBarPFull + 2;   // [2]
constexpr int kBarOFree = kBarOFull + 2;
constexpr int kNumBars = kBarOFree + 1;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffFlag = kOffTmemPtr + 4;
constexpr int kOffRed = (kOffFlag + 4 + 15) & ~15;  // float [2 buf][4 key quarters][64 heads]
constexpr int kOffSeq = kOffRed + 2 * 4 * 64 * 4;    // int32 [kMaxBatch] tiles per sequence, then prefix
constexpr int kOffML = kOffSeq + 2 * kMaxBatch * 4;  // float mloc[64], lloc[64], mrecv[64], lrecv[64]
constexpr int kSmemUsed = kOffML + 4 * 64 * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemS = 256;  // S^T buffer b: 128 lanes (keys) x 64 cols (heads) at 256 + 64 b
constexpr uint32_t kSoftmaxWarps = 8;
constexpr uint32_t kSmThreads = 32 * kSoftmaxWarps;
constexpr int kPartFloats = kH * kDv + 2 * kH;  // O, m (log2), l
constexpr size_t kPartBytes = sizeof(float) * kPartFloats;
constexpr size_t kCounterBytes = 4 * kMaxBatch;

struct DecodeParams {
  CUtensorMap q_map, k_map, v_map;
  const int32_t* seq_lens;
  int32_t batch, s, l, b, sparse, grid;
  int32_t pair;  // 1: cluster of 2 CTAs per sequence, halves of its tiles, merged through DSMEM
  int64_t t_cap;
  float scale_log2;
  void* o;
  int64_t o_sb, o_sh;
  int32_t out_bf16;
  float* lse;
  float* part;
  int32_t* counters;
  unsigned long long* trace;  // debug timeline of CTA 0 (NULL in production)
};

struct SeqTiles {
  int32_t n_sink, loc_begin, n_tiles;
  int32_t pos;  // query position p = seq_len - 1 (< 2^31)
};

__device__ __forceinline__ SeqTiles seq_tiles(const DecodeParams& p, int bi) {
  int64_t L = p.seq_lens[bi];
  L = L < 1 ? 1 : (L > p.t_cap ? p.t_cap : L);
  SeqTiles t;
  t.pos = (int32_t)(L - 1);
  const int32_t last_tile = t.pos >> 7;
  if (!p.sparse) {
    t.n_sink = 0;
    t.loc_begin = 0;
    t.n_tiles = last_tile + 1;
    return t;
  }
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

__global__ void __launch_bounds__(kThreads, 1) decode_tc_kernel(const __grid_constant__ DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  volatile int32_t* flag = reinterpret_cast<volatile int32_t*>(smem + kOffFlag);
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  int32_t* s_ntiles = reinterpret_cast<int32_t*>(smem + kOffSeq);
  int32_t* s_pref = s_ntiles + kMaxBatch;

  DTRACE(0, 0);
  // ---- tiles per sequence (parallel), prefix sums, this CTA's range of the flattened tile space
  for (int bi = threadIdx.x; bi < p.batch; bi += blockDim.x) s_ntiles[bi] = seq_tiles(p, bi).n_tiles;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int bi = 0; bi < p.batch; ++bi) {
      s_pref[bi] = (int32_t)acc;
      acc += s_ntiles[bi];
    }
    *flag = (int32_t)acc;
  }
  __syncthreads();
  const int64_t total = *flag;
  const int64_t G = p.grid, c = blockIdx.x;
  int64_t lo, hi;
  const uint32_t prank = p.pair ? cluster_ctarank() : 0;
  if (p.pair) {  // sequence c/2; CTA rank r takes half r of its tile list (rank 1 may get none)
    const int bi = (int)(c >> 1);
    const int64_t nt = s_ntiles[bi], mid = (nt + 1) / 2;
    lo = s_pref[bi] + (prank ? mid : 0);
    hi = s_pref[bi] + (prank ? nt : mid);
  } else {
    lo = c * total / G;
    hi = (c + 1) * total / G;
    if (lo >= hi) return;  // uniform across the CTA: nothing allocated yet
  }
  __syncthreads();  // everyone has read *flag before it is reused
  float* mloc = reinterpret_cast<float*>(smem + kOffML);
  float* lloc = mloc + 64;
  float* mrecv = mloc + 128;
  float* lrecv = mloc + 192;
  if (p.pair) {
    for (int i = threadIdx.x; i < 64; i += blockDim.x) {
      mloc[i] = -INFINITY;
      lloc[i] = 0.f;
    }
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar(kBarRingFull + i), 1);
      mbar_init(bar(kBarRingEmpty + i), 1);
    }
    mbar_init(bar(kBarQFull), 1);
    mbar_init(bar(kBarQEmpty), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), kSoftmaxWarps);
      mbar_init(bar(kBarPFull + i), kSoftmaxWarps);
      mbar_init(bar(kBarOFull + i), 1);
    }
    mbar_init(bar(kBarOFree), kSoftmaxWarps);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(&p.v_map);
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_ptr_smem), kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;
  DTRACE(0, 1);

  // first sequence touching [lo, hi): binary search on the prefix sums
  int b_first = p.pair ? (int)(c >> 1) : 0;
  if (!p.pair) {
    int lo_b = 0, hi_b = p.batch - 1;
    while (lo_b < hi_b) {
      const int mid = (lo_b + hi_b + 1) >> 1;
      if (s_pref[mid] <= lo) lo_b = mid;
      else hi_b = mid - 1;
    }
    b_first = lo_b;
  }
  // piece enumeration shared by all roles: sequence bi, local tiles [t0, t1)
  auto for_each_piece = [&](auto&& body) {
    for (int bi = b_first; bi < p.batch && s_pref[bi] < hi && lo < hi; ++bi) {
      const int64_t pref = s_pref[bi], nt = s_ntiles[bi];
      const int64_t a = pref > lo ? pref : lo, e = (pref + nt) < hi ? (pref + nt) : hi;
      if (a < e) body(bi, seq_tiles(p, bi), (int)(a - pref), (int)(e - pref), pref);
    }
  };

  if (warp == 0) {
    // ----------------------------------------------------- TMA producer (warp-uniform, elected lane issues)
    const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
    uint32_t stage = 0, phase = 0, pc = 0;
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
    for_each_piece([&](int bi, const SeqTiles& st, int t0, int t1, int64_t) {
      mbar_wait(bar(kBarQEmpty), (pc & 1) ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(bar(kBarQFull), kQBytes);
        for (int cc = 0; cc < kChunks; ++cc)
          tma_load_3d(sbase + kOffQ + cc * 8192, &p.q_map, cc * 64, 0, bi, bar(kBarQFull), pol_q);
      }
      __syncwarp();
      auto load_k = [&](int32_t k0) {
        for (int cc = 0; cc < kChunks; ++cc) {
          const uint32_t dst = acquire();
          if (elect_one()) {
            mbar_arrive_expect_tx(bar(kBarRingFull + stage), kStageBytes);
            tma_load_3d(dst, &p.k_map, cc * 64, k0, bi, bar(kBarRingFull + stage), pol_kv);
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
              mbar_arrive_expect_tx(bar(kBarRingFull + stage), kStageBytes);
              for (int e = 0; e < 4; ++e)
                tma_load_3d(dst + e * 4096, &p.v_map, 256 * nh + 64 * e, k0 + 32 * kq, bi, bar(kBarRingFull + stage),
                            pol_kv);
            }
            __syncwarp();
            next();
          }
      };
      load_k(tile_k0(st, t0));
      for (int i = t0 + 1; i < t1; ++i) {
        load_k(tile_k0(st, i));
        load_v(tile_k0(st, i - 1));
      }
      load_v(tile_k0(st, t1 - 1));
      ++pc;
    });
  } else if (warp == 1) {
    // ----------------------------------------------------- UMMA issuer (warp-uniform, elected lane issues)
    // Transposed products keep M = 128 (full-rate UMMA; M = 64 runs at half rate):
    //   S^T[key][head] = K Q^T : M = 128 keys (A = K chunk, K-major), N = 64 heads (B = Q chunk, K-major)
    //   O^T[dim][head] += V^T P : M = 128 dims (A = V slab, MN-major), N = 64 heads (B = P [key][head], MN-major)
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 64, true, true);
    const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
    const uint64_t dr_k = sdesc_sw128(sbase + kOffRing, 16, 1024);
    const uint64_t dr_v = sdesc_sw128(sbase + kOffRing, 4096, 1024);
    const uint64_t dp = sdesc_sw128(sbase + kOffP, 8192, 1024);
    uint32_t stage = 0, phase = 0, pc = 0, g = 0;
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
      for (int cc = 0; cc < kChunks; ++cc) {
        mbar_wait(bar(kBarRingFull + stage), phase);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_1sm(d, dr_k + (uint64_t)((kStageBytes * stage + 32 * k) >> 4),
                          dq + (uint64_t)((8192 * cc + 32 * k) >> 4), idesc_s, (cc | k) != 0);
          umma_commit_1sm(bar(kBarRingEmpty + stage));
        }
        __syncwarp();
        next();
      }
      if (elect_one()) umma_commit_1sm(bar(kBarSFull + buf));
      __syncwarp();
      DTRACE(2, gi);
    };
    auto issue_pv = [&](uint32_t gi, bool first) {
      const uint32_t buf = gi & 1;
      DTRACE(3, gi);
      mbar_wait(bar(kBarPFull + buf), (gi >> 1) & 1);
      if (first && pc > 0) mbar_wait(bar(kBarOFree), (pc - 1) & 1);
      DTRACE(4, gi);
      tc_fence_after();
      for (int kq = 0; kq < 4; ++kq)
        for (int nh = 0; nh < 2; ++nh) {
          mbar_wait(bar(kBarRingFull + stage), phase);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
              for (int dg = 0; dg < 2; ++dg)
                umma_bf16_1sm(tmem + 64 * (2 * nh + dg),
                              dr_v + (uint64_t)((kStageBytes * stage + 8192 * dg + 2048 * kk) >> 4),
                              dp + (uint64_t)((buf * kPBytes + (32 * kq + 16 * kk) * 128) >> 4), idesc_pv,
                              !(first && kq == 0 && kk == 0));
            umma_commit_1sm(bar(kBarRingEmpty + stage));
          }
          __syncwarp();
          next();
        }
      if (elect_one()) umma_commit_1sm(bar(kBarOFull + buf));
      __syncwarp();
      DTRACE(5, gi);
    };
    for_each_piece([&](int, const SeqTiles&, int t0, int t1, int64_t) {
      mbar_wait(bar(kBarQFull), pc & 1);
      tc_fence_after();
      const uint32_t g0 = g;
      const int n = t1 - t0;
      for (int i = 0; i < n; ++i) {
        issue_s(g0 + i);
        if (i == n - 1) {
          if (elect_one()) umma_commit_1sm(bar(kBarQEmpty));
          __syncwarp();
        }
        if (i >= 1) issue_pv(g0 + i - 1, i - 1 == 0);
      }
      issue_pv(g0 + n - 1, n == 1);
      g += n;
      ++pc;
    });
  } else {
    // ----------------------------------------------------- softmax / merge / epilogue (warps 2..9)
    // TMEM lane quarter wq = warp % 4: S^T lanes = keys 32 wq .. 32 wq + 31 of the tile, O^T lanes = dims
    // 128 g + 32 wq + lane. Column half ch = (warp - 2) / 4 selects heads [32 ch, 32 ch + 32): a thread holds one
    // key's (or one dim's) 32 heads. Per-head maxima over keys: redux.sync.max.f32 within the warp, then the
    // 4 key-quarter warps through shared memory.
    const uint32_t wq = warp & 3;
    const uint32_t ch = (warp - 2) >> 2;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const float sl2 = p.scale_log2;
    const float ln2 = 0.69314718055994531f;
    const int tid = (int)threadIdx.x - 64;  // 0..255
    uint32_t g = 0, pc = 0;
    for_each_piece([&](int bi, const SeqTiles& st, int t0, int t1, int64_t pref) {
      float m_used[32], lpart[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        m_used[j] = -INFINITY;
        lpart[j] = 0.f;
      }
      const int n = t1 - t0;
      for (int i = 0; i < n; ++i) {
        const uint32_t gi = g + i, buf = gi & 1;
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
        // per-head max over this warp's 32 keys (masked keys excluded), then over the 4 key quarters
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
      // -------- end of piece: l[h] = sum over the 128 key lanes of lpart[h]
      const uint32_t gl = g + n - 1;
      mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
      if (warp == 2) DTRACE(9, pc);
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
      const float lh = (ls[32 * ch + lane] + ls[64 + 32 * ch + lane]) + (ls[128 + 32 * ch + lane] + ls[192 + 32 * ch + lane]);
      named_bar_sync(1, kSmThreads);
      const bool whole = (t0 == 0 && t1 == st.n_tiles);
      if (p.pair) {  // the DSMEM merge after the role loop needs (m, l) per head; O stays in TMEM
        if (wq == 0) {
          mloc[32 * ch + lane] = m_used_lane(m_used, lane);
          lloc[32 * ch + lane] = lh;
        }
        g += n;
        ++pc;
        return;
      }
      // per-head (l, m) for this thread's 32 heads: shuffle from lane j
      float inv_l[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) inv_l[j] = 1.0f / __shfl_sync(0xffffffffu, lh, j);
      if (whole) {
#pragma unroll 1
        for (int gg = 0; gg < 4; ++gg) {
          uint32_t ov[32];
          tmem_ld32(taddr + 64 * gg + 32 * ch, ov);
          tmem_wait_ld();
          const int dim = 128 * gg + 32 * (int)wq + (int)lane;
          char* ob = reinterpret_cast<char*>(p.o) +
                     ((int64_t)bi * p.o_sb + (int64_t)(32 * ch) * p.o_sh + dim) * (p.out_bf16 ? 2 : 4);
          const int64_t hstride = p.o_sh * (p.out_bf16 ? 2 : 4);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float val = __uint_as_float(ov[j]) * inv_l[j];
            if (p.out_bf16) {
              const uint32_t u = pack_bf16x2(val, 0.f) & 0xFFFFu;
              *reinterpret_cast<unsigned short*>(ob + j * hstride) = (unsigned short)u;
            } else {
              *reinterpret_cast<float*>(ob + j * hstride) = val;
            }
          }
        }
        if (p.lse && wq == 0) {
          const float lj = lh;  // lane j holds head 32 ch + j
          p.lse[(int64_t)bi * kH + 32 * ch + lane] = (m_used_lane(m_used, lane) + __log2f(lj)) * ln2;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar(kBarOFree));
      } else {
        // partial of piece (c, bi) -> slot c + bi, layout [head][dim] + m[64] + l[64]
        float* slot = p.part + (size_t)(c + bi) * kPartFloats;
#pragma unroll 1
        for (int gg = 0; gg < 4; ++gg) {
          uint32_t ov[32];
          tmem_ld32(taddr + 64 * gg + 32 * ch, ov);
          tmem_wait_ld();
          const int dim = 128 * gg + 32 * (int)wq + (int)lane;
#pragma unroll
          for (int j = 0; j < 32; ++j) slot[(size_t)(32 * ch + j) * kDv + dim] = __uint_as_float(ov[j]);
        }
        if (wq == 0) {
          slot[kH * kDv + 32 * ch + lane] = m_used_lane(m_used, lane);
          slot[kH * kDv + kH + 32 * ch + lane] = lh;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar(kBarOFree));
        const int64_t first_tile = pref, last_tile_g = pref + st.n_tiles - 1;
        const int64_t c_first = ((first_tile + 1) * G - 1) / total;
        const int64_t c_last = ((last_tile_g + 1) * G - 1) / total;
        auto nonempty = [&](int64_t cc) { return (cc * total) / G < ((cc + 1) * total) / G; };
        if (warp == 2) DTRACE(10, pc);
        __threadfence();
        named_bar_sync(1, kSmThreads);
        if (tid == 0) {
          int npieces = 0;
          for (int64_t cp = c_first; cp <= c_last; ++cp) npieces += nonempty(cp) ? 1 : 0;
          const int old = atomicAdd(&p.counters[bi], 1);
          *flag = (old == npieces - 1) ? 1 : 0;
        }
        named_bar_sync(1, kSmThreads);
        if (*flag) {
          __threadfence();
          // merge in CTA order (deterministic): thread -> (head row = tid / 4, 128 dims at 128 (tid % 4))
          const int row = tid >> 2, dim_base = 128 * (tid & 3);
          float mt = -INFINITY;
          for (int64_t cp = c_first; cp <= c_last; ++cp)
            if (nonempty(cp)) mt = fmaxf(mt, __ldcg(p.part + (size_t)(cp + bi) * kPartFloats + kH * kDv + row));
          float lt = 0.f;
          for (int64_t cp = c_first; cp <= c_last; ++cp) {
            if (!nonempty(cp)) continue;
            const float* sl = p.part + (size_t)(cp + bi) * kPartFloats;
            lt += __ldcg(sl + kH * kDv + kH + row) * ex2(__ldcg(sl + kH * kDv + row) - mt);
          }
          const float inv = 1.0f / lt;
          char* obase = reinterpret_cast<char*>(p.o) +
                        ((int64_t)bi * p.o_sb + (int64_t)row * p.o_sh + dim_base) * (p.out_bf16 ? 2 : 4);
#pragma unroll 1
          for (int d0 = 0; d0 < 128; d0 += 32) {
            float acc[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = 0.f;
            for (int64_t cp = c_first; cp <= c_last; ++cp) {
              if (!nonempty(cp)) continue;
              const float* sl = p.part + (size_t)(cp + bi) * kPartFloats;
              const float w = ex2(__ldcg(sl + kH * kDv + row) - mt) * inv;
              const float4* src = reinterpret_cast<const float4*>(sl + (size_t)row * kDv + dim_base + d0);
              float4 a4[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) a4[j] = __ldcg(src + j);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                acc[4 * j] = fmaf(w, a4[j].x, acc[4 * j]);
                acc[4 * j + 1] = fmaf(w, a4[j].y, acc[4 * j + 1]);
                acc[4 * j + 2] = fmaf(w, a4[j].z, acc[4 * j + 2]);
                acc[4 * j + 3] = fmaf(w, a4[j].w, acc[4 * j + 3]);
              }
            }
            if (p.out_bf16) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                st_global_v4(obase + 2 * (d0 + 8 * j), pack_bf16x2(acc[8 * j], acc[8 * j + 1]),
                             pack_bf16x2(acc[8 * j + 2], acc[8 * j + 3]), pack_bf16x2(acc[8 * j + 4], acc[8 * j + 5]),
                             pack_bf16x2(acc[8 * j + 6], acc[8 * j + 7]));
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                st_global_v4(obase + 4 * (d0 + 4 * j), __float_as_uint(acc[4 * j]), __float_as_uint(acc[4 * j + 1]),
                             __float_as_uint(acc[4 * j + 2]), __float_as_uint(acc[4 * j + 3]));
            }
          }
          if (p.lse && (tid & 3) == 0) p.lse[(int64_t)bi * kH + row] = (mt + __log2f(lt)) * ln2;
          if (tid == 0) p.counters[bi] = 0;  // self-reset for the next launch
          if (warp == 2) DTRACE(11, pc);
        }
        named_bar_sync(1, kSmThreads);  // *flag is read by all before the next piece may rewrite it
      }
      g += n;
      ++pc;
    });
  }
  __syncwarp();
  if (p.pair) {
    // ---- merge the two halves of sequence c/2 through distributed shared memory. CTA r finalises heads
    // [32 r, 32 r + 32): warps with ch != r send their heads' O^T (fp32, thread-major swizzled 512-B rows) and
    // (m, l) into the partner's idle ring; warps with ch == r combine. Ring and P are idle: all tiles done.
    const int bi = (int)(c >> 1);
    const uint32_t partner = prank ^ 1;
    const bool has_tiles = lo < hi;
    tc_fence_before();
    cluster_sync();  // #1: both CTAs finished their tiles (and wrote mloc / lloc)
    tc_fence_after();
    if (warp >= 2 && warp <= 9) {
      const uint32_t wq = warp & 3, ch = (warp - 2) >> 2;
      const uint32_t taddr = tmem + ((wq * 32) << 16);
      const uint32_t t = wq * 32 + lane;  // thread-major row in the receive buffer (128 rows x 512 B)
      if (ch != prank) {
        const uint32_t rbuf = mapa(sbase + kOffRing, partner);
#pragma unroll 1
        for (int gg = 0; gg < 4; ++gg) {
          uint32_t ov[32];
          if (has_tiles) {
            tmem_ld32(taddr + 64 * gg + 32 * ch, ov);
            tmem_wait_ld();
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] = 0u;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t k16 = (uint32_t)(gg * 8 + q);  // 16-byte chunk index of this thread's row
            st_cluster_v4(rbuf + t * 512 + ((k16 ^ (t & 31)) << 4), ov[4 * q], ov[4 * q + 1], ov[4 * q + 2],
                          ov[4 * q + 3]);
          }
        }
        if (wq == 0) {
          st_cluster_f32(mapa(smem_u32(mrecv + 32 * ch + lane), partner), mloc[32 * ch + lane]);
          st_cluster_f32(mapa(smem_u32(lrecv + 32 * ch + lane), partner), lloc[32 * ch + lane]);
        }
      }
    }
    cluster_sync();  // #2: partner data landed
    if (warp == 2) DTRACE(10, 0);
    if (warp >= 2 && warp <= 9) {
      const uint32_t wq = warp & 3, ch = (warp - 2) >> 2;
      if (ch == prank) {
        const uint32_t taddr = tmem + ((wq * 32) << 16);
        const uint32_t t = wq * 32 + lane;
        float w_own[32], w_par[32], inv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int h = 32 * ch + j;
          const float mo = mloc[h], mp = mrecv[h], lo_ = lloc[h], lp = lrecv[h];
          const float mt = fmaxf(mo, mp);
          w_own[j] = lo_ > 0.f ? ex2(mo - mt) : 0.f;
          w_par[j] = lp > 0.f ? ex2(mp - mt) : 0.f;
          inv[j] = 1.0f / (w_own[j] * lo_ + w_par[j] * lp);
        }
        const char* rb = reinterpret_cast<const char*>(smem + kOffRing);
#pragma unroll 1
        for (int gg = 0; gg < 4; ++gg) {
          uint32_t ov[32];
          if (has_tiles) {
            tmem_ld32(taddr + 64 * gg + 32 * ch, ov);
            tmem_wait_ld();
          }
          float pv[32];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t k16 = (uint32_t)(gg * 8 + q);
            const float4 f = *reinterpret_cast<const float4*>(rb + t * 512 + ((k16 ^ (t & 31)) << 4));
            pv[4 * q] = f.x;
            pv[4 * q + 1] = f.y;
            pv[4 * q + 2] = f.z;
            pv[4 * q + 3] = f.w;
          }
          const int dim = 128 * gg + 32 * (int)wq + (int)lane;
          uint8_t* stg = smem + kOffQ;  // Q is idle now: stage O [32 heads][512 dims]
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float own = (has_tiles && w_own[j] > 0.f) ? __uint_as_float(ov[j]) * w_own[j] : 0.f;
            const float val = fmaf(pv[j], w_par[j], own) * inv[j];
            if (p.out_bf16)
              *reinterpret_cast<unsigned short*>(stg + (j * kDv + dim) * 2) = (unsigned short)(pack_bf16x2(val, 0.f) & 0xFFFFu);
            else
              *reinterpret_cast<float*>(stg + (j * kDv + dim) * 4) = val;
          }
        }
        named_bar_sync(2, 128);  // the 4 combining warps
        {
          const int esz = p.out_bf16 ? 2 : 4, row_bytes = kDv * esz, chunks = 32 * row_bytes / 16;
          const uint8_t* stg = smem + kOffQ;
          for (int k = (int)t; k < chunks; k += 128) {
            const int j = (k * 16) / row_bytes, off = (k * 16) % row_bytes;
            const uint4 w = *reinterpret_cast<const uint4*>(stg + j * row_bytes + off);
            char* dst = reinterpret_cast<char*>(p.o) + ((int64_t)bi * p.o_sb + (int64_t)(32 * ch + j) * p.o_sh) * esz + off;
            st_global_v4(dst, w.x, w.y, w.z, w.w);
          }
        }
        if (p.lse && wq == 0) {
          const int h = 32 * ch + lane;
          const float mo = mloc[h], mp = mrecv[h], mt = fmaxf(mo, mp);
          const float lt = (lloc[h] > 0.f ? lloc[h] * ex2(mo - mt) : 0.f) + (lrecv[h] > 0.f ? lrecv[h] * ex2(mp - mt) : 0.f);
          p.lse[(int64_t)bi * kH + h] = (mt + __log2f(lt)) * 0.69314718055994531f;
        }
      }
    }
  }
  if (warp == 2) DTRACE(11, 0);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, kTmemCols);
  }
}

bool decode_pair_mode(const AttnProblem& a, int sms) { return a.sparse && 2 * (int64_t)a.batch <= sms; }

int64_t decode_grid(const AttnProblem& a, int sms) {
  // SSA: a CTA pair per sequence (DSMEM merge) while 2B CTAs fit in one wave, else one CTA per sequence
  if (decode_pair_mode(a, sms)) return 2 * (int64_t)a.batch;
  if (a.sparse && 4 * (int64_t)a.batch >= sms) return a.batch < sms ? a.batch : sms;
  if (a.sparse) {
    const int64_t tmax = ((int64_t)a.s + a.l) * a.b / 128;  // tiles per sequence at most
    const int64_t total = tmax * a.batch;
    const int64_t per = (total + sms - 1) / sms;
    return (total + per - 1) / per;
  }
  return sms;
}

}  // namespace

size_t decode_ws_bytes_unused(const AttnProblem& a) {
  const int64_t G = decode_grid(a, device_sm_count());
  return kCounterBytes + (size_t)(G + a.batch) * kPartBytes;
}

unsigned long long* g_pair_trace = nullptr;

cudaError_t launch_decode_pair(const AttnProblem& a, cudaStream_t st) {
  if (a.heads != kH) return cudaErrorNotSupported;
  if (a.batch > kMaxBatch) return cudaErrorNotSupported;
  if (a.n_kv >= (1ll << 31)) return cudaErrorNotSupported;
  DecodeParams p;
  memset(&p, 0, sizeof(p));
  p.seq_lens = a.seq_lens;
  p.batch = a.batch;
  p.s = a.s;
  p.l = a.l;
  p.b = a.sparse ? a.b : 128;
  p.sparse = a.sparse;
  p.t_cap = a.n_kv;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.o = a.o;
  p.o_sb = a.o_sb;
  p.o_sh = a.o_sh;
  p.out_bf16 = a.out_bf16;
  p.lse = a.lse;
  p.trace = g_pair_trace;
  const int sms = device_sm_count();
  p.grid = 2 * a.batch;
  p.counters = nullptr;  // pair mode: no global partials
  p.part = nullptr;
  const KvSeg& s = a.kv.seg[0];
  if (!encode_3d(&p.q_map, a.q, kDqk, kH, a.batch, a.q_sh, a.q_sb, 64)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.k_map, s.k, kDqk, (uint64_t)a.n_kv, a.batch, s.k_st, s.k_sb, 128)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.v_map, s.v, kDv, (uint64_t)a.n_kv, a.batch, s.v_st, s.v_sb, 32)) return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  p.pair = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemAlloc;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = p.pair ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, decode_tc_kernel, p);
  if (le != cudaSuccess) return le;
  count_launch();
  return cudaGetLastError();
}

bool decode_pair_eligible(const AttnProblem& a, int sms) {
  return a.sparse && a.heads == kH && a.b % 128 == 0 && 2 * (int64_t)a.batch <= sms && a.n_kv < (1ll << 31) &&
         a.batch <= kMaxBatch;
}

}  // namespace loza

extern "C" void loza_debug_set_pair_trace(void* dev_ptr) { loza::g_pair_trace = (unsigned long long*)dev_ptr; }
