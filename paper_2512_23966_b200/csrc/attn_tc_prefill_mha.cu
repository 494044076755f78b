// tcgen05 bf16 SSA prefill in the non-absorbed (MHA) form: per head q_h, k_h of d_qk = 192
// (128 nope + 64 RoPE) and v_h of d_v = 128 (the window up-projected per head), Eq. 4 with the same block
// selection as the absorbed kernel. Derived from attn_tc_prefill.cu (same pipeline):
//  * Work unit = 128 query tokens of one (batch, head); CTA r of the pair owns tokens 64 r .. 64 r + 63. An S tile
//    is 256 keys = two selected 128-key sub-blocks (CTA r stages sub-block 2i + r as its half of the UMMA B
//    operand). S = Q K^T: 12 UMMAs M128 N256 K16 (A = resident Q, 24 KB/SM); online softmax in registers (8
//    warps, a row's 256 logits in 4 threads, lazy rescale); P (bf16) to SMEM; O += P V: 16 UMMAs M128 N128 K16
//    (cta_group::2: CTA r holds V dims [64 r, 64 r + 64) for all 256 keys). TMEM: O 64 cols, S 2 x 128 cols.
//  * Loads: 5-D TMA views {64, tokens, chunks, heads, batch} (the per-head strides); one ring of 4 x 32 KB slots
//    in UMMA order (K(0), K(1), V(0), K(2), V(1), ...): a K item is 128 keys x dims [0, 128) (2 chunks), the
//    RoPE chunk [128, 192) rides a one-slot ring, a V item is the tile's 256 keys x 64 dims (two boxes). Warp 0
//    issues Q and K items, warp 10 V items, with the position handshake of the absorbed kernel.
//  * Epilogue: O -> registers (O released) -> bf16 -> two [64 x 64] swizzled boxes in the idle P buffer -> TMA
//    tensor stores (one round); fp32 output with plain stores.
#include <math.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {
using namespace sm100;

#define FULL_L(slot) (full_l + 8 * (slot))
#define QFULL_L(c) (qfull_l + 8 * (c))
constexpr int kDqk = 192, kDv = 128, kChunks = 3;
constexpr int kThreads = 352;  // warp 0 Q/K TMA, warp 1 MMA, warps 2-9 softmax/epilogue, warp 10 V TMA
constexpr int kVWarp = 10;
constexpr int kSlots = 4;
constexpr int kSlotBytes = 32768;
constexpr int kChunkBytes = 16384;  // 128 keys x 64 dims
constexpr int kKItems = 1;          // big-ring K items per tile: chunks {0,1}; chunk 2 via the one-slot ring
constexpr int kVItems = 1;          // V items per tile: 256 keys x this CTA's 64 dims
constexpr int kQBytes = kChunks * 64 * 128;  // 24576 per CTA
constexpr int kPBytes = 4 * 64 * 128;        // 32768: 4 key chunks (64 keys) x 64 rows
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffRing = kOffP + kPBytes;
constexpr int kOffRope = kOffRing + kSlots * kSlotBytes;
constexpr int kOffBar = kOffRope + kChunkBytes;
constexpr int kBarFull = 0;
constexpr int kBarEmpty = kBarFull + kSlots;
constexpr int kBarRopeFull = kBarEmpty + kSlots;
constexpr int kBarRopeEmpty = kBarRopeFull + 1;
constexpr int kBarQFull = kBarRopeEmpty + 1;     // [3]
constexpr int kBarQEmpty = kBarQFull + kChunks;  // [3]
constexpr int kBarSFull = kBarQEmpty + kChunks;  // [2]
constexpr int kBarSFree = kBarSFull + 2;         // [2]
constexpr int kBarPFull = kBarSFree + 2;         // [1]
constexpr int kBarOFull = kBarPFull + 1;         // [2]
constexpr int kBarOFree = kBarOFull + 2;
constexpr int kNumBars = kBarOFree + 1;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffPub = kOffTmemPtr + 4;
constexpr int kOffRed = (kOffPub + 8 + 15) & ~15;
constexpr int kSmemUsed = kOffRed + 2 * 4 * 64 * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 0, kTmemS = 256;  // S buffer b at 256 + 128 b
constexpr uint32_t kSoftmaxWarps = 8;
constexpr uint32_t kArrivalsPerPair = 2 * kSoftmaxWarps;

struct MhaParams {
  CUtensorMap q_map;   // 5-D, box 64 tokens x 1 chunk
  CUtensorMap k1_map;  // 5-D, box 128 keys x 1 chunk (the RoPE chunk 2)
  CUtensorMap k2_map;  // 5-D, box 128 keys x 2 chunks
  CUtensorMap v_map;   // 5-D, box 128 keys x 1 chunk
  CUtensorMap o_map;   // 5-D, box 64 tokens x 1 chunk (bf16 output)
  int32_t batch, n_q, heads;
  int64_t q_start, n_kv;
  int32_t s, l, b, sparse, causal;
  float scale_log2;
  void* o;
  int64_t o_sb, o_st, o_sh;
  int32_t out_bf16;
  float* lse;
  int64_t units_per_bh, total_units;
};

struct Unit {
  int32_t bi, h;           // batch, head
  int64_t row0;            // first query token of the unit (local index)
  int64_t tok_lo, tok_hi;  // absolute positions
  int32_t n_sink, loc_begin, n128, n_tiles;
};

__device__ __forceinline__ Unit make_unit(const MhaParams& p, int64_t u) {
  Unit U;
  const int64_t bh = u / p.units_per_bh;
  U.bi = (int32_t)(bh / p.heads);
  U.h = (int32_t)(bh - (int64_t)U.bi * p.heads);
  U.row0 = (u - bh * p.units_per_bh) * 128;
  int64_t rlast = U.row0 + 127;
  if (rlast > p.n_q - 1) rlast = p.n_q - 1;
  U.tok_lo = p.q_start + U.row0;
  U.tok_hi = p.q_start + rlast;
  const int64_t last_sub = p.causal ? U.tok_hi / 128 : (p.n_kv - 1) / 128;
  if (!p.sparse) {
    U.n_sink = 0;
    U.loc_begin = 0;
    U.n128 = (int32_t)(last_sub + 1);
  } else {
    const int64_t tpb = p.b / 128, QB = U.tok_lo / p.b;
    int64_t sink_end = (QB + 1 < p.s ? QB + 1 : p.s) * tpb;
    if (sink_end > last_sub + 1) sink_end = last_sub + 1;
    int64_t lb = QB - p.l + 1;
    if (lb < p.s) lb = p.s;
    lb *= tpb;
    int64_t le = (QB + 1) * tpb;
    if (le > last_sub + 1) le = last_sub + 1;
    U.n_sink = (int32_t)sink_end;
    U.loc_begin = (int32_t)lb;
    U.n128 = (int32_t)(sink_end + (le > lb ? le - lb : 0));
  }
  U.n_tiles = (U.n128 + 1) / 2;
  return U;
}
__device__ __forceinline__ int64_t sub_k0(const Unit& U, int j) {
  if (j >= U.n128) return -1;
  return (int64_t)(j < U.n_sink ? j : U.loc_begin + (j - U.n_sink)) * 128;
}
// key row coordinate of a sub-block; a missing sub-block maps to an out-of-bounds box (zeros)
__device__ __forceinline__ int32_t kv_row(const MhaParams& p, int64_t k0) { return k0 < 0 ? (int32_t)p.n_kv : (int32_t)k0; }
__device__ __forceinline__ int64_t unit_index(const MhaParams& p, int64_t it) { return p.total_units - 1 - it; }

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    prefill_mha_kernel(const __grid_constant__ MhaParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* red = reinterpret_cast<float*>(smem + kOffRed);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSlots; ++i) {
      mbar_init(bar(kBarFull + i), 1);
      mbar_init(bar(kBarEmpty + i), 1);
    }
    mbar_init(bar(kBarRopeFull), 1);
    mbar_init(bar(kBarRopeEmpty), 1);
    for (int i = 0; i < kChunks; ++i) {
      mbar_init(bar(kBarQFull + i), 1);
      mbar_init(bar(kBarQEmpty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), kArrivalsPerPair);
      mbar_init(bar(kBarOFull + i), 1);
    }
    mbar_init(bar(kBarPFull), kArrivalsPerPair);
    mbar_init(bar(kBarOFree), kArrivalsPerPair);
    reinterpret_cast<volatile uint32_t*>(smem + kOffPub)[0] = 0;
    reinterpret_cast<volatile uint32_t*>(smem + kOffPub)[1] = 0;
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.k1_map);
    prefetch_tmap(&p.k2_map);
    prefetch_tmap(&p.v_map);
  }
  if (warp == 1) tmem_alloc<2>(smem_u32(tmem_ptr_smem), kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;

  const int64_t n_iter_total = p.total_units;
  const int64_t ncl = nclusters_x();
  const int64_t cid = cluster_id_x();

  struct RingPos {
    uint32_t slot = 0, phase = 0, pos = 0;
    __device__ __forceinline__ void step() {
      ++pos;
      if (++slot == kSlots) {
        slot = 0;
        phase ^= 1;
      }
    }
    __device__ __forceinline__ void skip(int n) {
      for (int i = 0; i < n; ++i) step();
    }
  };
  // producers' position handshake (see attn_tc_prefill.cu: parity waits on a shared ring alias otherwise)
  volatile uint32_t* pub = reinterpret_cast<volatile uint32_t*>(smem + kOffPub);
  auto acquire = [&](const RingPos& rp, int me) {
    if (lane == 0) pub[me] = rp.pos;
    if (rp.pos >= (uint32_t)kSlots)
      while (pub[me ^ 1] <= rp.pos - kSlots) {
      }
    __syncwarp();
    mbar_wait(bar(kBarEmpty + rp.slot), rp.phase ^ 1);
  };
  if (warp == 0) {
    // ===================================================== Q + K items producer (both CTAs)
    const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
    const uint32_t full_l = mapa(bar(kBarFull), 0), qfull_l = mapa(bar(kBarQFull), 0),
                   rope_l = mapa(bar(kBarRopeFull), 0);
    const uint32_t ring = sbase + kOffRing;
    RingPos rp;
    uint32_t uc = 0, gk = 0;
    auto load_k = [&](const Unit& U, int i) {
      const int32_t row = kv_row(p, sub_k0(U, 2 * i + (int)rank));  // CTA r stages sub-block 2i+r
      mbar_wait(bar(kBarRopeEmpty), (gk & 1) ^ 1);
      if (elect_one()) {
        if (rank == 0) mbar_arrive_expect_tx(bar(kBarRopeFull), 2 * kChunkBytes);
        tma_load_5d_pair(sbase + kOffRope, &p.k1_map, 0, row, 2, U.h, U.bi, rope_l, pol_kv);
      }
      __syncwarp();
      for (int j = 0; j < kKItems; ++j, rp.step()) {
        acquire(rp, 0);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + rp.slot), 2 * kSlotBytes);
          tma_load_5d_pair(ring + rp.slot * kSlotBytes, &p.k2_map, 0, row, 2 * j, U.h, U.bi, FULL_L(rp.slot), pol_kv);
        }
        __syncwarp();
      }
      ++gk;
    };
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = make_unit(p, unit_index(p, it));
      if (lane == 0) pub[0] = rp.pos;
      __syncwarp();
      for (int c = 0; c < kChunks; ++c) {
        mbar_wait(bar(kBarQEmpty + c), (uc & 1) ^ 1);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarQFull + c), 2 * 8192);
          tma_load_5d_pair(sbase + kOffQ + c * 8192, &p.q_map, 0, (int32_t)(U.row0 + 64 * rank), c, U.h, U.bi,
                           QFULL_L(c), pol_q);
        }
        __syncwarp();
      }
      load_k(U, 0);
      for (int i = 1; i < U.n_tiles; ++i) {
        load_k(U, i);
        rp.skip(kVItems);  // V(i-1): warp kVWarp
      }
      rp.skip(kVItems);
    }
    if (lane == 0) pub[0] = 0xFFFFFFFFu;
  } else if (warp == kVWarp) {
    // ===================================================== V items producer (both CTAs)
    const uint64_t pol_kv = policy_evict_last();
    const uint32_t full_l = mapa(bar(kBarFull), 0);
    const uint32_t ring = sbase + kOffRing;
    RingPos rp;
    auto load_v = [&](const Unit& U, int i) {
      acquire(rp, 1);
      if (elect_one()) {
        if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + rp.slot), 2 * kSlotBytes);
        // keys of sub-blocks A, B (128 each), this CTA's dim chunk r
        for (int kg = 0; kg < 2; ++kg)
          tma_load_5d_pair(ring + rp.slot * kSlotBytes + kg * kChunkBytes, &p.v_map, 0,
                           kv_row(p, sub_k0(U, 2 * i + kg)), (int)rank, U.h, U.bi, FULL_L(rp.slot), pol_kv);
      }
      __syncwarp();
      rp.step();
    };
    for (int64_t it = cid; it < n_iter_total; it += ncl) {
      const Unit U = make_unit(p, unit_index(p, it));
      rp.skip(kKItems);
      for (int i = 1; i < U.n_tiles; ++i) {
        rp.skip(kKItems);
        load_v(U, i - 1);
      }
      load_v(U, U.n_tiles - 1);
    }
    if (lane == 0) pub[1] = 0xFFFFFFFFu;
  } else if (warp == 1) {
    // ===================================================== MMA issuer (leader CTA only)
    if (rank == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 256, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, false, true);
      const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
      const uint64_t dk = sdesc_sw128(sbase + kOffRing, 16, 1024);
      const uint64_t dp = sdesc_sw128(sbase + kOffP, 16, 1024);
      const uint64_t dv = sdesc_sw128(sbase + kOffRing, 16, 1024);  // [256 keys][64 dims] MN-major (one 64-dim atom)
      uint32_t uc = 0, g = 0;
      RingPos rp;
      auto issue_s = [&](uint32_t gi, bool first, bool last) {
        const uint32_t buf = gi & 1;
        mbar_wait(bar(kBarSFree + buf), ((gi >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + kTmemS + 128 * buf;
        for (int j = 0; j <= kKItems; ++j) {  // big item (chunks 0, 1), then the RoPE chunk 2
          const bool rope = j == kKItems;
          const uint32_t slot = rp.slot;
          const int nc = rope ? 1 : 2;
          if (first) {
            mbar_wait(bar(kBarQFull + 2 * j), uc & 1);
            if (nc == 2) mbar_wait(bar(kBarQFull + 2 * j + 1), uc & 1);
          }
          if (rope)
            mbar_wait(bar(kBarRopeFull), gi & 1);
          else
            mbar_wait(bar(kBarFull + slot), rp.phase);
          tc_fence_after();
          const uint32_t kaddr = rope ? (uint32_t)(kOffRope - kOffRing) : kSlotBytes * slot;
          if (elect_one()) {
            for (int cc = 0; cc < nc; ++cc) {
              const int c = 2 * j + cc;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                umma_bf16_pair(d, dq + (uint64_t)((8192 * c + 32 * k) >> 4),
                               dk + (uint64_t)((kaddr + kChunkBytes * cc + 32 * k) >> 4), idesc_s, (c | k) != 0);
            }
            umma_commit_pair_mc(bar(rope ? kBarRopeEmpty : kBarEmpty + slot), 3);
            if (last) {
              umma_commit_pair_mc(bar(kBarQEmpty + 2 * j), 3);
              if (nc == 2) umma_commit_pair_mc(bar(kBarQEmpty + 2 * j + 1), 3);
            }
          }
          __syncwarp();
          if (!rope) rp.step();
        }
        if (elect_one()) umma_commit_pair_mc(bar(kBarSFull + buf), 3);
        __syncwarp();
      };
      auto issue_pv = [&](uint32_t gi, bool first) {
        mbar_wait(bar(kBarPFull), gi & 1);
        if (first && uc > 0) mbar_wait(bar(kBarOFree), (uc - 1) & 1);
        tc_fence_after();
        const uint32_t slot = rp.slot;
        mbar_wait(bar(kBarFull + slot), rp.phase);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 16; ++kk) {
            const int key = 16 * kk;  // key of the 256-key tile (P column)
            umma_bf16_pair(tmem + kTmemO, dp + (uint64_t)((8192 * (key >> 6) + 2 * (key & 63)) >> 4),
                           dv + (uint64_t)((kSlotBytes * slot + 2048 * kk) >> 4), idesc_pv, !(first && kk == 0));
          }
          umma_commit_pair_mc(bar(kBarEmpty + slot), 3);
        }
        __syncwarp();
        rp.step();
        if (elect_one()) umma_commit_pair_mc(bar(kBarOFull + (gi & 1)), 3);
        __syncwarp();
      };
      for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
        const Unit U = make_unit(p, unit_index(p, it));
        const uint32_t g0 = g;
        for (int i = 0; i < U.n_tiles; ++i) {
          issue_s(g0 + i, i == 0, i == U.n_tiles - 1);
          if (i >= 1) issue_pv(g0 + i - 1, i - 1 == 0);
        }
        issue_pv(g0 + U.n_tiles - 1, U.n_tiles == 1);
        g += U.n_tiles;
      }
    }
  } else {
    // ===================================================== softmax + epilogue (warps 2..9, both CTAs)
    // S: lane tl holds row r = tl % 64 and the 128 logits of sub-block kh = tl / 64; warps with ch take 64 of them.
    // O (N = 128, 2x2 fold): lanes 0-63 hold dims [0, 64) of their row, lanes 64-127 dims [64, 128); a warp
    // with ch holds 32 of those 64 (columns [32 ch, 32 ch + 32)).
    const uint32_t wq = warp & 3;
    const uint32_t ch = (warp - 2) >> 2;
    const uint32_t tl = wq * 32 + lane;
    const uint32_t r = tl & 63, kh = tl >> 6, q4 = 2 * kh + ch;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const uint32_t sfree0 = mapa(bar(kBarSFree), 0), pfull = mapa(bar(kBarPFull), 0), ofree = mapa(bar(kBarOFree), 0);
    const float ln2 = 0.69314718055994531f;
    const float sl2 = p.scale_log2;
    const int causal = p.causal;
    const int64_t n_kv = p.n_kv;
    constexpr uint32_t kSmThreads = 32 * kSoftmaxWarps;
    uint32_t g = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl) {
      const Unit U = make_unit(p, unit_index(p, it));
      const int64_t row_g = U.row0 + 64 * rank + r;  // local query token
      const bool row_ok = row_g < p.n_q;
      const int64_t my_tok = p.q_start + (row_ok ? row_g : p.n_q - 1);
      float m_used = -INFINITY, lrow = 0.f;
      for (int i = 0; i < U.n_tiles; ++i) {
        const uint32_t gi = g + i, buf = gi & 1;
        const int64_t kb0 = sub_k0(U, 2 * i + (int)kh);
        int32_t nvalid = 64;
        if (kb0 < 0) {
          nvalid = 0;
        } else {
          const int64_t c0 = kb0 + 64 * ch;
          int64_t lim = n_kv - c0;
          if (causal && my_tok + 1 - c0 < lim) lim = my_tok + 1 - c0;
          nvalid = lim < 0 ? 0 : (lim > 64 ? 64 : (int32_t)lim);
        }
        mbar_wait(bar(kBarSFull + buf), (gi >> 1) & 1);
        tc_fence_after();
        const uint32_t sa = taddr + kTmemS + 128 * buf + 64 * ch;
        uint32_t v[64];
        tmem_ld32(sa, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(sfree0 + 8 * buf);
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
        float* rb = red + buf * 256;
        rb[q4 * 64 + r] = tmax;
        named_bar_sync(1, kSmThreads);
        tmax = fmaxf(fmaxf(rb[r], rb[64 + r]), fmaxf(rb[128 + r], rb[192 + r]));
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
        if (i > 0) {
          const uint32_t gp = gi - 1;
          mbar_wait(bar(kBarOFull + (gp & 1)), (gp >> 1) & 1);
          tc_fence_after();
          if (__any_sync(0xffffffffu, resc)) {
            uint32_t ov[32];
            tmem_ld32(taddr + kTmemO + 32 * ch, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
            tmem_st32(taddr + kTmemO + 32 * ch, ov);
            tmem_wait_st();
          }
        }
        const uint32_t prow = sbase + kOffP + q4 * 8192 + r * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          st_shared_v4(prow + ((u ^ (r & 7)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        lrow = lrow * corr + ((ps0 + ps1) + (ps2 + ps3));
        m_used = m_new;
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(pfull);
      }
      // ---------------- epilogue: O / l -> global (this thread: row r, dims 64 kh + 32 ch + [0, 32))
      const uint32_t gl = g + U.n_tiles - 1;
      mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
      tc_fence_after();
      float* ls = red + ((gl + 1) & 1) * 256;
      ls[q4 * 64 + r] = lrow;
      named_bar_sync(1, kSmThreads);
      const float ltot = (ls[r] + ls[64 + r]) + (ls[128 + r] + ls[192 + r]);
      const float inv = 1.0f / ltot;
      named_bar_sync(1, kSmThreads);
      uint32_t ov[32];
      tmem_ld32(taddr + kTmemO + 32 * ch, ov);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ofree);
      const int dim0 = 64 * (int)kh + 32 * (int)ch;
      if (p.out_bf16) {
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          w[j] = pack_bf16x2(__uint_as_float(ov[2 * j]) * inv, __uint_as_float(ov[2 * j + 1]) * inv);
        // box kh = dims [64 kh, +64): row r at kh * 8192 + 128 r, 16-B units 4 ch + q swizzled by r & 7
        const uint32_t box = sbase + kOffP + kh * 8192 + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_shared_v4(box + (((4 * ch + q) ^ (r & 7)) << 4), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
        fence_proxy_async_smem();
        named_bar_sync(1, kSmThreads);
        if (warp == 2 && lane == 0) {
          for (int m = 0; m < 2; ++m)
            tma_store_5d(&p.o_map, sbase + kOffP + m * 8192, 0, (int32_t)(U.row0 + 64 * rank), m, U.h, U.bi);
          bulk_commit_group();
          bulk_wait_group_read0();  // staging (the P buffer) is rewritten by the next unit's first softmax
        }
        named_bar_sync(1, kSmThreads);
      } else if (row_ok) {
        float* dst = reinterpret_cast<float*>(p.o) + (int64_t)U.bi * p.o_sb + row_g * p.o_st + (int64_t)U.h * p.o_sh + dim0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_global_v4(dst + 4 * q, __float_as_uint(__uint_as_float(ov[4 * q]) * inv),
                       __float_as_uint(__uint_as_float(ov[4 * q + 1]) * inv),
                       __float_as_uint(__uint_as_float(ov[4 * q + 2]) * inv),
                       __float_as_uint(__uint_as_float(ov[4 * q + 3]) * inv));
      }
      if (p.lse && row_ok && q4 == 0)
        p.lse[((int64_t)U.bi * p.heads + U.h) * p.n_q + row_g] = (m_used + __log2f(ltot)) * ln2;
      g += U.n_tiles;
    }
    if (warp == 2 && lane == 0) bulk_wait_group0();
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

cudaError_t launch_prefill_mha(const AttnProblem& a, int64_t k_sh, int64_t v_sh, cudaStream_t st) {
  if (a.d_qk != kDqk || a.d_v != kDv) return cudaErrorNotSupported;
  MhaParams p;
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
  p.o_st = a.o_st;
  p.o_sh = a.o_sh;
  p.out_bf16 = a.out_bf16;
  p.lse = a.lse;
  p.units_per_bh = (a.n_q + 127) / 128;
  p.total_units = p.units_per_bh * a.batch * a.heads;
  if (p.total_units == 0) return cudaSuccess;
  const KvSeg& s = a.kv.seg[0];
  const uint64_t H = (uint64_t)a.heads;
  if (!encode_5d_heads(&p.q_map, a.q, kDqk, (uint64_t)a.n_q, H, a.batch, a.q_st, a.q_sh, a.q_sb, 64, 1) ||
      !encode_5d_heads(&p.k1_map, s.k, kDqk, (uint64_t)a.n_kv, H, a.batch, s.k_st, k_sh, s.k_sb, 128, 1) ||
      !encode_5d_heads(&p.k2_map, s.k, kDqk, (uint64_t)a.n_kv, H, a.batch, s.k_st, k_sh, s.k_sb, 128, 2) ||
      !encode_5d_heads(&p.v_map, s.v, kDv, (uint64_t)a.n_kv, H, a.batch, s.v_st, v_sh, s.v_sb, 128, 1))
    return cudaErrorInvalidValue;
  if (a.out_bf16 && !encode_5d_heads(&p.o_map, a.o, kDv, (uint64_t)a.n_q, H, a.batch, a.o_st, a.o_sh, a.o_sb, 64, 1))
    return cudaErrorInvalidValue;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(prefill_mha_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int sms = device_sm_count();
  int64_t ncl = sms / 2;
  if (ncl > p.total_units) ncl = p.total_units;
  prefill_mha_kernel<<<(unsigned)(2 * ncl), kThreads, kSmemAlloc, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza
