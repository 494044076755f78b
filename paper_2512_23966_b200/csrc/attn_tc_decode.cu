// tcgen05 bf16 split-KV decode over the latent MLA cache (d_qk 576, d_v 512, H = 64):
// SSA decode (Eq. 4 at p = seq_len - 1: sink block(s) + the last l blocks) and the
// full-attention decode comparator (Eq. 1 over [0, seq_len)).
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
constexpr int kMaxBatch = 1024;
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
constexpr int kOffRed = (kOffFlag + 4 + 15) & ~15;  // float [2 buf][2 ch][64]; end of piece reuses it
constexpr int kOffSeq = kOffRed + 2 * 2 * 64 * 4;    // int32 [kMaxBatch] tiles per sequence, then prefix
constexpr int kSmemUsed = kOffSeq + 2 * kMaxBatch * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemS = 256;
constexpr uint32_t kSoftmaxWarps = 8;
constexpr uint32_t kSmThreads = 32 * kSoftmaxWarps;
constexpr int kPartFloats = kH * kDv + 2 * kH;  // O, m (log2), l
constexpr size_t kPartBytes = sizeof(float) * kPartFloats;
constexpr size_t kCounterBytes = 4 * kMaxBatch;

struct DecodeParams {
  CUtensorMap q_map, k_map, v_map;
  const int32_t* seq_lens;
  int32_t batch, s, l, b, sparse, grid;
  int64_t t_cap;
  float scale_log2;
  void* o;
  int64_t o_sb, o_sh;
  int32_t out_bf16;
  float* lse;
  float* part;
  int32_t* counters;
  int32_t* status;            // LOZA_ERR_SHAPE when a seq_len was outside [1, t_cap] (clamped)
  unsigned long long* trace;  // debug timeline of CTA 0 (NULL in production)
};

struct SeqTiles {
  int32_t n_sink, loc_begin, n_tiles;
  int32_t pos;  // query position p = seq_len - 1 (< 2^31)
};

__device__ __forceinline__ SeqTiles seq_tiles(const DecodeParams& p, int bi) {
  int64_t L = p.seq_lens[bi];
  if ((L < 1 || L > p.t_cap) && p.status) *p.status = LOZA_ERR_SHAPE;
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
  const int64_t lo = c * total / G, hi = (c + 1) * total / G;
  if (lo >= hi) return;  // uniform across the CTA: nothing allocated yet
  __syncthreads();       // everyone has read *flag before it is reused

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
  int b_first = 0;
  {
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
    for (int bi = b_first; bi < p.batch && s_pref[bi] < hi; ++bi) {
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
    constexpr uint32_t idesc_s = idesc_bf16_f32(64, 128, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(64, 256, false, true);
    const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
    const uint64_t dr_k = sdesc_sw128(sbase + kOffRing, 16, 1024);
    const uint64_t dr_v = sdesc_sw128(sbase + kOffRing, 4096, 1024);
    const uint64_t dp = sdesc_sw128(sbase + kOffP, 16, 1024);
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
      const uint32_t d = tmem + kTmemS + 128 * buf;
      for (int cc = 0; cc < kChunks; ++cc) {
        mbar_wait(bar(kBarRingFull + stage), phase);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_1sm(d, dq + (uint64_t)((8192 * cc + 32 * k) >> 4),
                          dr_k + (uint64_t)((kStageBytes * stage + 32 * k) >> 4), idesc_s, (cc | k) != 0);
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
              umma_bf16_1sm(tmem + ((uint32_t)(16 * nh) << 16),
                            dp + (uint64_t)((buf * kPBytes + (kq >> 1) * 8192 + (kq & 1) * 64 + kk * 32) >> 4),
                            dr_v + (uint64_t)((kStageBytes * stage + 2048 * kk) >> 4), idesc_pv,
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
    // TMEM sub-partition wq = warp % 4 holds heads 16 wq .. 16 wq + 15: S and O[:, 0:256) in lanes 0-15,
    // O[:, 256:512) in lanes 16-31. Warps 2-5 (ch = 0) take logit columns [0, 64) and O columns [0, 128);
    // warps 6-9 (ch = 1) columns [64, 128) and O columns [128, 256).
    const uint32_t wq = warp & 3;
    const uint32_t ch = (warp - 2) >> 2;
    const uint32_t half = lane >> 4;
    const uint32_t row = wq * 16 + (lane & 15);  // head
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const float sl2 = p.scale_log2;
    const float ln2 = 0.69314718055994531f;
    const int tid = (int)threadIdx.x - 64;  // 0..255
    uint32_t g = 0, pc = 0;
    for_each_piece([&](int bi, const SeqTiles& st, int t0, int t1, int64_t pref) {
      float m_used = -INFINITY, lrow = 0.f;
      const int n = t1 - t0;
      for (int i = 0; i < n; ++i) {
        const uint32_t gi = g + i, buf = gi & 1;
        const int32_t c0 = tile_k0(st, t0 + i) + 64 * (int32_t)ch;
        int32_t nvalid = st.pos + 1 - c0;  // keys <= pos among this warp's 64 columns
        nvalid = nvalid < 0 ? 0 : (nvalid > 64 ? 64 : nvalid);
        if (warp == 2) DTRACE(6, gi);
        mbar_wait(bar(kBarSFull + buf), (gi >> 1) & 1);
        if (warp == 2) DTRACE(7, gi);
        tc_fence_after();
        uint32_t v[64];
        const uint32_t sa = taddr + kTmemS + 128 * buf + 64 * ch;
        tmem_ld32(sa, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar(kBarSFree + buf));
        if (nvalid < 64) {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j >= nvalid) v[j] = __float_as_uint(-INFINITY);
        }
        float mx0 = __uint_as_float(v[0]), mx1 = __uint_as_float(v[1]), mx2 = __uint_as_float(v[2]),
              mx3 = __uint_as_float(v[3]);
#pragma unroll
        for (int j = 4; j < 64; j += 4) {
          mx0 = fmaxf(mx0, __uint_as_float(v[j]));
          mx1 = fmaxf(mx1, __uint_as_float(v[j + 1]));
          mx2 = fmaxf(mx2, __uint_as_float(v[j + 2]));
          mx3 = fmaxf(mx3, __uint_as_float(v[j + 3]));
        }
        float tmax = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * sl2;
        float* rb = red + buf * 128;
        if (half == 0) rb[ch * 64 + row] = tmax;
        named_bar_sync(1, kSmThreads);
        tmax = fmaxf(rb[row], rb[64 + row]);  // lanes 16-31: the same head's value (their S reads were unused)
        const bool resc = tmax > m_used + 8.0f;
        const float m_new = resc ? tmax : m_used;
        const float corr = resc ? ex2(m_used - m_new) : 1.0f;
        float ps0 = 0.f, ps1 = 0.f, ps2 = 0.f, ps3 = 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float e0 = ex2(fmaf(__uint_as_float(v[2 * j]), sl2, -m_new));
          const float e1 = ex2(fmaf(__uint_as_float(v[2 * j + 1]), sl2, -m_new));
          const float e2 = ex2(fmaf(__uint_as_float(v[2 * j + 2]), sl2, -m_new));
          const float e3 = ex2(fmaf(__uint_as_float(v[2 * j + 3]), sl2, -m_new));
          ps0 += e0;
          ps1 += e1;
          ps2 += e2;
          ps3 += e3;
          pk[j] = pack_bf16x2(e0, e1);
          pk[j + 1] = pack_bf16x2(e2, e3);
        }
        if (half == 0) {
          const uint32_t prow = sbase + kOffP + buf * kPBytes + ch * 8192 + row * 128;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            st_shared_v4(prow + ((u ^ (row & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        if (i > 0) {
          const uint32_t gp = gi - 1;
          mbar_wait(bar(kBarOFull + (gp & 1)), (gp >> 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, resc)) {
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {  // O columns [128 ch, +128), both lane halves
              uint32_t ov[32];
              tmem_ld32(taddr + 128 * ch + 32 * cc, ov);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
              tmem_st32(taddr + 128 * ch + 32 * cc, ov);
            }
            tmem_wait_st();
          }
        }
        lrow = lrow * corr + ((ps0 + ps1) + (ps2 + ps3));
        m_used = m_new;
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar(kBarPFull + buf));
        if (warp == 2) DTRACE(8, gi);
      }
      // -------- end of piece: combine the two column halves' sums, then write O or a partial
      const uint32_t gl = g + n - 1;
      mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
      if (warp == 2) DTRACE(9, pc);
      tc_fence_after();
      float* ls = red + ((gl + 1) & 1) * 128;
      if (half == 0) ls[ch * 64 + row] = lrow;
      named_bar_sync(1, kSmThreads);
      const float l_row = ls[row] + ls[64 + row];
      const float m_row = m_used;  // identical in both lane halves and both column halves
      named_bar_sync(1, kSmThreads);
      const bool whole = (t0 == 0 && t1 == st.n_tiles);
      const int dim_base = 256 * (int)half + 128 * (int)ch;
      if (whole) {
        const float inv = 1.0f / l_row;
        char* obase = reinterpret_cast<char*>(p.o) +
                      ((int64_t)bi * p.o_sb + (int64_t)row * p.o_sh + dim_base) * (p.out_bf16 ? 2 : 4);
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t ov[32];
          tmem_ld32(taddr + 128 * ch + 32 * cc, ov);
          tmem_wait_ld();
          if (p.out_bf16) {
            uint32_t w[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              w[j] = pack_bf16x2(__uint_as_float(ov[2 * j]) * inv, __uint_as_float(ov[2 * j + 1]) * inv);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_global_v4(obase + 64 * cc + 16 * q, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              st_global_v4(obase + 128 * cc + 16 * q, __float_as_uint(__uint_as_float(ov[4 * q]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 1]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 2]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 3]) * inv));
          }
        }
        if (p.lse && half == 0 && ch == 0) p.lse[(int64_t)bi * kH + row] = (m_row + __log2f(l_row)) * ln2;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar(kBarOFree));
      } else {
        // partial of piece (c, bi) -> slot c + bi
        float* slot = p.part + (size_t)(c + bi) * kPartFloats;
        float* orow = slot + (size_t)row * kDv + dim_base;
#pragma unroll 1
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t ov[32];
          tmem_ld32(taddr + 128 * ch + 32 * cc, ov);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 8; ++q)
            st_global_v4(orow + 32 * cc + 4 * q, ov[4 * q], ov[4 * q + 1], ov[4 * q + 2], ov[4 * q + 3]);
        }
        if (half == 0 && ch == 0) {
          slot[kH * kDv + row] = m_row;
          slot[kH * kDv + kH + row] = l_row;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar(kBarOFree));
        // pieces of this sequence: the non-empty CTAs among [c_first, c_last]
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
          // merge in CTA order (deterministic); thread -> (head row, 128 dims at dim_base)
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
          if (p.lse && half == 0 && ch == 0) p.lse[(int64_t)bi * kH + row] = (mt + __log2f(lt)) * ln2;
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
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, kTmemCols);
  }
}

int64_t decode_grid(const AttnProblem& a, int sms) {
  // SSA: one CTA per sequence (no split, no merge) once the batch fills a quarter of the SMs
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

// decode workspace: [0, 256) status word (int32 at 0) + reserved, then (flattened kernel only) the per-sequence
// counters and the split partials
size_t decode_tc_ws_bytes(const AttnProblem& a) {
  const int sms = device_sm_count();
  if (decode_coop_eligible(a, sms) || decode_ks_eligible(a, sms)) return kDecodeStatusBytes;
  const int64_t G = decode_grid(a, sms);
  return kDecodeStatusBytes + kCounterBytes + (size_t)(G + a.batch) * kPartBytes;
}

unsigned long long* g_decode_trace = nullptr;

cudaError_t launch_decode_tc(const AttnProblem& a, void* ws, size_t ws_bytes, cudaStream_t st) {
  int32_t* status = ws && ws_bytes >= kDecodeStatusBytes ? reinterpret_cast<int32_t*>(ws) : nullptr;
  cudaError_t pe;
  if (decode_pair_dispatch(a, status, st, &pe)) return pe;
  if (a.ring) return cudaErrorNotSupported;  // the ring cache is read by the key-split pair kernel only
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
  p.trace = g_decode_trace;
  const int sms = device_sm_count();
  p.grid = (int32_t)decode_grid(a, sms);
  if (ws_bytes < kDecodeStatusBytes + kCounterBytes + (size_t)(p.grid + a.batch) * kPartBytes)
    return cudaErrorInvalidValue;
  p.status = status;
  p.counters = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + kDecodeStatusBytes);
  p.part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + kDecodeStatusBytes + kCounterBytes);
  const KvSeg& s = a.kv.seg[0];
  if (!encode_3d(&p.q_map, a.q, kDqk, kH, a.batch, a.q_sh, a.q_sb, 64)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.k_map, s.k, kDqk, (uint64_t)a.n_kv, a.batch, s.k_st, s.k_sb, 128)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.v_map, s.v, kDv, (uint64_t)a.n_kv, a.batch, s.v_st, s.v_sb, 32)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
  if (e != cudaSuccess) return e;
  decode_tc_kernel<<<p.grid, kThreads, kSmemAlloc, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza

extern "C" void loza_debug_set_decode_trace(void* dev_ptr) { loza::g_decode_trace = (unsigned long long*)dev_ptr; }
