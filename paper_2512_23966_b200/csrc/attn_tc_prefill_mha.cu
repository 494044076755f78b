// tcgen05 bf16 SSA prefill in the non-absorbed (MHA) form: per head q_h, k_h of d_qk = 192
// (128 nope + 64 RoPE) and v_h of d_v = 128 (the window up-projected per head), Eq. 4 with the same block
// selection as the absorbed kernel (attn_tc_prefill.cu), re-shaped for the smaller head:
//  * Work unit = 256 query tokens of one (batch, head) on a CTA pair; CTA r owns tokens 128 r .. 128 r + 127, one
//    per TMEM lane (no fold). A tile is one selected 128-key sub-block: S = Q K^T as 12 UMMAs cta_group::2
//    M256 N128 K16 (A = resident Q, 48 KB/SM; CTA r stages keys 64 r .. 64 r + 63 of the sub-block), online
//    softmax in registers (8 warps: a row's 128 logits in 2 threads of a warp pair, lazy rescale), P (bf16) to
//    SMEM, O += P V as 8 UMMAs M256 N128 K16 (CTA r stages V dims 64 r .. 64 r + 63). M256 keeps every UMMA at
//    64 tensor cycles (an M128 N128 pair UMMA is 32: issue-bound) and halves the K/V bytes per flop
//    (40 KB per SM per tile). TMEM: O 128 cols, S 2 x 128 cols.
//  * A unit spans up to two query blocks (b = 128): it walks the union of their windows (the sink blocks and
//    local blocks max(s, QB_lo - l + 1) .. QB_hi) and each row masks keys outside its own window (Eq. 4's
//    block set) - for (1,7,128) 9 sub-blocks where a row needs 8.
//  * Loads: 5-D TMA views {64, tokens, chunks, heads, batch}; one ring of 6 x 24 KB slots in UMMA order
//    (K(0), K(1), V(0), K(2), V(1), ...): a K item is 64 keys x 192 dims (3 chunks, one box), a V item 128 keys x
//    64 dims. Warp 0 issues Q and K items, warp 10 V items, with the absorbed kernel's position handshake.
//  * Epilogue: O -> registers (O released) -> bf16 -> two [128 x 64] swizzled boxes in the idle P buffer -> TMA
//    tensor stores (each box written and stored by the 4 warps of its column half); fp32 output: plain stores.
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
// warpgroup 0: warp 0 Q/K TMA, warp 1 MMA, warp 2 V TMA (64 regs); warpgroups 1-2: softmax (warps 4-11,
// 176 regs); warpgroup 3: epilogue (warps 12-15, 96 regs) -- setmaxnreg rebalances the 128/thread launch
constexpr int kThreads = 512;
constexpr int kVWarp = 2;
constexpr int kSmWarp0 = 4, kEpiWarp0 = 12;
constexpr int kSlots = 5;
constexpr int kSlotBytes = 24576;
constexpr int kKItemBytes = 64 * 128 * kChunks;  // 64 keys x 192 dims
constexpr int kVItemBytes = 128 * 128;           // 128 keys x 64 dims
constexpr int kQChunkBytes = 128 * 128;          // 128 rows x 64 dims
constexpr int kQBytes = kChunks * kQChunkBytes;  // 48 KB per buffer, 2 buffers (unit parity)
constexpr int kOffQ = 0;
constexpr int kOffRing = kOffQ + 2 * kQBytes;
constexpr int kOffBar = kOffRing + kSlots * kSlotBytes;
constexpr int kBarFull = 0;
constexpr int kBarEmpty = kBarFull + kSlots;
constexpr int kBarQFull = kBarEmpty + kSlots;        // [2][3]
constexpr int kBarQEmpty = kBarQFull + 2 * kChunks;  // [2][3]
constexpr int kBarSFull = kBarQEmpty + 2 * kChunks;  // [2]
constexpr int kBarPFull = kBarSFull + 2;             // [1]
constexpr int kBarOFull = kBarPFull + 1;             // [2] (tile parity)
constexpr int kBarOFree = kBarOFull + 2;             // [2] (O buffer = unit parity)
constexpr int kBarStageFree = kBarOFree + 2;         // [2] (Q buffer = unit parity; local, 1 store issuer)
constexpr int kBarOLast = kBarStageFree + 2;         // [2] a unit's last PV landed (O buffer parity)
constexpr int kBarLFull = kBarOLast + 2;             // [2] softmax -> epilogue: row sums and maxima (local)
constexpr int kBarLFree = kBarLFull + 2;             // [2] epilogue has read them (local)
constexpr int kUSlots = 4;                           // decoded-unit ring (scheduler warp -> every role)
constexpr int kBarUFull = kBarLFree + 2;             // [kUSlots]
constexpr int kBarUEmpty = kBarUFull + kUSlots;      // [kUSlots]
constexpr int kNumBars = kBarUEmpty + kUSlots;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffPub = kOffTmemPtr + 4;
constexpr int kOffRed = (kOffPub + 8 + 15) & ~15;
constexpr int kOffLs = kOffRed + 2 * 2 * 128 * 4;  // float lsum[2 ob][2 ch][128], mrow[2 ob][128]
constexpr int kOffU = kOffLs + (2 * 2 * 128 + 2 * 128) * 4;  // int32 [kUSlots][8]: bi, h, row0, n_sink, loc_begin, n_tiles
constexpr int kSmemUsed = kOffU + kUSlots * 8 * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 0, kTmemS = 256;  // O buffer ob at 128 ob, S buffer b at 256 + 128 b (P(b) in its cols 0-63)
constexpr uint32_t kSoftmaxWarps = 8;
#ifndef MHA_POLY_PAIRS
#define MHA_POLY_PAIRS 0x00000000u  // v5: 0% measured 1.316 ms vs 1.322 (25%), 1.34 (31%), 1.37 (50%)
#endif
constexpr uint32_t kPolyPairs = MHA_POLY_PAIRS;  // exp pairs (of 32 per thread and tile) computed by polynomial
constexpr uint32_t kArrivalsPerPair = 2 * kSoftmaxWarps;
constexpr uint32_t kEpiArrivalsPerPair = 2 * 4;

struct MhaParams {
  CUtensorMap q_map;  // 5-D, box 128 tokens x 1 chunk
  CUtensorMap k_map;  // 5-D, box 64 keys x 3 chunks
  CUtensorMap v_map;  // 5-D, box 128 keys x 1 chunk
  CUtensorMap o_map;  // 5-D, box 128 tokens x 1 chunk (bf16 output)
  int32_t batch, n_q, heads;
  int64_t q_start, n_kv;
  int32_t s, l, b, sparse, causal;
  float scale_log2;
  void* o;
  int64_t o_sb, o_st, o_sh;
  int32_t out_bf16;
  float* lse;
  uint32_t units_per_bh, total_units;
  FastDiv div_upb, div_heads, div_b;
  unsigned long long* trace;  // debug timeline (cluster 0, leader CTA, first 64 tiles), NULL in production
};

struct Unit {
  int32_t bi, h;           // batch, head
  int64_t row0;            // first query token of the unit (local index)
  int64_t tok_lo, tok_hi;  // absolute positions
  int32_t n_sink, loc_begin, n_tiles;
};

__device__ __forceinline__ Unit make_unit(const MhaParams& p, uint32_t u) {
  Unit U;  // 32-bit index math (64-bit division is a long software sequence on the unit-boundary path)
  const uint32_t bh = p.div_upb.div(u);
  U.bi = (int32_t)p.div_heads.div(bh);
  U.h = (int32_t)(bh - (uint32_t)U.bi * (uint32_t)p.heads);
  U.row0 = (int64_t)(u - bh * p.units_per_bh) * 256;
  int64_t rlast = U.row0 + 255;
  if (rlast > p.n_q - 1) rlast = p.n_q - 1;
  U.tok_lo = p.q_start + U.row0;
  U.tok_hi = p.q_start + rlast;
  const int64_t last_sub = p.causal ? U.tok_hi >> 7 : (p.n_kv - 1) >> 7;
  if (!p.sparse) {
    U.n_sink = 0;
    U.loc_begin = 0;
    U.n_tiles = (int32_t)(last_sub + 1);
  } else {
    // union over the unit's query blocks QB_lo..QB_hi of {sink blocks} + {local blocks} (in 128-key sub-blocks)
    const int64_t tpb = p.b >> 7, QB_lo = p.div_b.div((uint32_t)U.tok_lo), QB_hi = p.div_b.div((uint32_t)U.tok_hi);
    int64_t sink_end = (int64_t)p.s * tpb;
    if (sink_end > last_sub + 1) sink_end = last_sub + 1;
    int64_t lb = QB_lo - p.l + 1;
    if (lb < p.s) lb = p.s;
    lb *= tpb;
    int64_t le = (QB_hi + 1) * tpb;
    if (le > last_sub + 1) le = last_sub + 1;
    U.n_sink = (int32_t)sink_end;
    U.loc_begin = (int32_t)lb;
    U.n_tiles = (int32_t)(sink_end + (le > lb ? le - lb : 0));
  }
  return U;
}
__device__ __forceinline__ int64_t sub_k0(const Unit& U, int j) {
  return (int64_t)(j < U.n_sink ? j : U.loc_begin + (j - U.n_sink)) * 128;
}
__device__ __forceinline__ uint32_t unit_index(const MhaParams& p, int64_t it) { return p.total_units - 1 - (uint32_t)it; }

#define MTRACE(slot, idx) \
  if (p.trace && cid == 0 && rank == 0 && (idx) < 64 && lane == 0) p.trace[(slot)*64 + (idx)] = clock64();

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
    for (int i = 0; i < 2 * kChunks; ++i) {
      mbar_init(bar(kBarQFull + i), 1);
      mbar_init(bar(kBarQEmpty + i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarOFull + i), 1);
      mbar_init(bar(kBarOFree + i), kEpiArrivalsPerPair);
      mbar_init(bar(kBarStageFree + i), 1);
      mbar_init(bar(kBarOLast + i), 1);
      mbar_init(bar(kBarLFull + i), kSoftmaxWarps);
      mbar_init(bar(kBarLFree + i), 4);
    }
    for (int i = 0; i < kUSlots; ++i) {
      mbar_init(bar(kBarUFull + i), 1);
      // consumers: warps 0 and 2 (producers), 4-11 (softmax), 12-15 (epilogue), and the leader's MMA warp
      mbar_init(bar(kBarUEmpty + i), cluster_ctarank() == 0 ? 15 : 14);
    }
    mbar_init(bar(kBarPFull), kArrivalsPerPair);
    reinterpret_cast<volatile uint32_t*>(smem + kOffPub)[0] = 0;
    reinterpret_cast<volatile uint32_t*>(smem + kOffPub)[1] = 0;
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(&p.v_map);
    prefetch_tmap(&p.o_map);
  }
  if (warp == 1) tmem_alloc<2>(smem_u32(tmem_ptr_smem), kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;

  const int64_t n_iter_total = p.total_units;
  const int64_t ncl = nclusters_x();
  const int64_t cid = cluster_id_x();
  // the k-th unit of this cluster, decoded by the scheduler warp (warp 3) into the ring; every consumer warp
  // reads it and releases the slot (no 64-bit / multi-step index math on the MMA and softmax paths)
  volatile int32_t* uring = reinterpret_cast<volatile int32_t*>(smem + kOffU);
  auto get_unit = [&](uint32_t k) {
    const uint32_t slot = k % kUSlots;
    mbar_wait(bar(kBarUFull + slot), (k / kUSlots) & 1);
    Unit U;
    const volatile int32_t* e = uring + 8 * slot;
    U.bi = e[0];
    U.h = e[1];
    U.row0 = e[2];
    U.n_sink = e[3];
    U.loc_begin = e[4];
    U.n_tiles = e[5];
    U.tok_lo = U.tok_hi = 0;
    __syncwarp();
    if (lane == 0) mbar_arrive_local(bar(kBarUEmpty + slot));
    return U;
  };

  // All roles walk one continuous tile stream across this cluster's units: ring order K(0), K(1), V(0), K(2),
  // V(1), ... with no break at unit boundaries, so S of a unit's first tile is issued before the previous
  // unit's last PV (whose P waits on the softmax) and the tensor pipe does not drain between units.
  struct RingPos {
    uint32_t slot = 0, phase = 0, pos = 0;
    __device__ __forceinline__ void step() {
      ++pos;
      if (++slot == kSlots) {
        slot = 0;
        phase ^= 1;
      }
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
  if (warp < kSmWarp0) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
  if (warp == 0) {
    // ===================================================== Q + K items producer (both CTAs)
    const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
    const uint32_t full_l = mapa(bar(kBarFull), 0), qfull_l = mapa(bar(kBarQFull), 0);
    const uint32_t ring = sbase + kOffRing;
    RingPos rp;
    uint32_t uc = 0, g = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = get_unit(uc);
      const uint32_t qb = uc & 1, qpar = ((uc >> 1) & 1) ^ 1;
      if (lane == 0) pub[0] = rp.pos;
      __syncwarp();
      mbar_wait(bar(kBarStageFree + qb), qpar);  // the epilogue of unit uc - 2 staged its output here
      for (int c = 0; c < kChunks; ++c) {
        mbar_wait(bar(kBarQEmpty + kChunks * qb + c), qpar);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarQFull + kChunks * qb + c), 2 * kQChunkBytes);
          tma_load_5d_pair(sbase + kOffQ + kQBytes * qb + c * kQChunkBytes, &p.q_map, 0,
                           (int32_t)(U.row0 + 128 * rank), c, U.h, U.bi, QFULL_L(kChunks * qb + c), pol_q);
        }
        __syncwarp();
      }
      for (int i = 0; i < U.n_tiles; ++i, ++g) {
        acquire(rp, 0);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + rp.slot), 2 * kKItemBytes);
          tma_load_5d_pair(ring + rp.slot * kSlotBytes, &p.k_map, 0, (int32_t)(sub_k0(U, i) + 64 * rank), 0, U.h,
                           U.bi, FULL_L(rp.slot), pol_kv);
        }
        __syncwarp();
        rp.step();
        if (g > 0) rp.step();  // V(g - 1): warp kVWarp
      }
    }
    if (lane == 0) pub[0] = 0xFFFFFFFFu;
  } else if (warp == kVWarp) {
    // ===================================================== V items producer (both CTAs)
    const uint64_t pol_kv = policy_evict_last();
    const uint32_t full_l = mapa(bar(kBarFull), 0);
    const uint32_t ring = sbase + kOffRing;
    RingPos rp;
    int32_t pv_row = -1, pv_h = 0, pv_b = 0;  // the tile whose V comes next
    auto load_v = [&]() {
      acquire(rp, 1);
      if (elect_one()) {
        if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + rp.slot), 2 * kVItemBytes);
        tma_load_5d_pair(ring + rp.slot * kSlotBytes, &p.v_map, 0, pv_row, (int)rank, pv_h, pv_b, FULL_L(rp.slot),
                         pol_kv);
      }
      __syncwarp();
      rp.step();
    };
    uint32_t vk = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++vk) {
      const Unit U = get_unit(vk);
      for (int i = 0; i < U.n_tiles; ++i) {
        rp.step();  // K(g)
        if (pv_row >= 0) load_v();
        pv_row = (int32_t)sub_k0(U, i);
        pv_h = U.h;
        pv_b = U.bi;
      }
    }
    if (pv_row >= 0) load_v();
    if (lane == 0) pub[1] = 0xFFFFFFFFu;
  } else if (warp == 1) {
    // ===================================================== MMA issuer (leader CTA only)
    if (rank == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(256, 128, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(256, 128, false, true);
      const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
      const uint64_t dk = sdesc_sw128(sbase + kOffRing, 16, 1024);
      const uint64_t dv = sdesc_sw128(sbase + kOffRing, 16, 1024);  // [128 keys][64 dims] MN-major (one atom wide)
      uint32_t g = 0, uc = 0;
      RingPos rp;
      auto issue_s = [&](uint32_t gi, uint32_t u, bool first, bool last) {
        const uint32_t buf = gi & 1, qb = u & 1;
        MTRACE(0, gi);
        // S buffer buf was last read by PV(gi - 2) (its P), issued before this S: the in-order tensor pipe
        // finishes that read before these writes; its S was consumed before PFull(gi - 2)
        const uint32_t slot = rp.slot;
        mbar_wait(bar(kBarFull + slot), rp.phase);
        tc_fence_after();
        MTRACE(1, gi);
        const uint32_t d = tmem + kTmemS + 128 * buf;
        for (int c = 0; c < kChunks; ++c) {
          if (first) {
            mbar_wait(bar(kBarQFull + kChunks * qb + c), (u >> 1) & 1);
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16_pair(d, dq + (uint64_t)((kQBytes * qb + kQChunkBytes * c + 32 * k) >> 4),
                             dk + (uint64_t)((kSlotBytes * slot + 8192 * c + 32 * k) >> 4), idesc_s, (c | k) != 0);
            if (last) umma_commit_pair_mc(bar(kBarQEmpty + kChunks * qb + c), 3);
          }
          __syncwarp();
        }
        if (elect_one()) {
          umma_commit_pair_mc(bar(kBarEmpty + slot), 3);
          umma_commit_pair_mc(bar(kBarSFull + buf), 3);
        }
        __syncwarp();
        MTRACE(2, gi);
        rp.step();
      };
      // PV of tile gi of unit u (first: the unit's first tile, overwrites O buffer u & 1)
      auto issue_pv = [&](uint32_t gi, uint32_t u, bool first, bool last) {
        const uint32_t ob = u & 1;
        MTRACE(3, gi);
        mbar_wait(bar(kBarPFull), gi & 1);
        MTRACE(4, gi);
        if (first && u >= 2) mbar_wait(bar(kBarOFree + ob), ((u >> 1) & 1) ^ 1);
        const uint32_t slot = rp.slot;
        mbar_wait(bar(kBarFull + slot), rp.phase);
        tc_fence_after();
        MTRACE(5, gi);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int key = 16 * kk;  // key of the 128-key tile (P column)
            umma_bf16_pair_ts(tmem + kTmemO + 128 * ob, tmem + kTmemS + 128 * (gi & 1) + key / 2,
                              dv + (uint64_t)((kSlotBytes * slot + 2048 * kk) >> 4), idesc_pv, !(first && kk == 0));
          }
          umma_commit_pair_mc(bar(kBarEmpty + slot), 3);
          umma_commit_pair_mc(bar(kBarOFull + (gi & 1)), 3);
          if (last) umma_commit_pair_mc(bar(kBarOLast + ob), 3);
        }
        __syncwarp();
        rp.step();
      };
      uint32_t pv_u = 0;
      bool pv_first = false, pv_last = false, have_pv = false;
      for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
        const Unit U = get_unit(uc);
        for (int i = 0; i < U.n_tiles; ++i, ++g) {
          issue_s(g, uc, i == 0, i == U.n_tiles - 1);
          if (have_pv) issue_pv(g - 1, pv_u, pv_first, pv_last);
          have_pv = true;
          pv_u = uc;
          pv_first = i == 0;
          pv_last = i == U.n_tiles - 1;
        }
      }
      if (have_pv) issue_pv(g - 1, pv_u, pv_first, pv_last);
    }
  } else if (warp == 3) {
    // ===================================================== unit scheduler (both CTAs)
    uint32_t k = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++k) {
      const uint32_t slot = k % kUSlots;
      mbar_wait(bar(kBarUEmpty + slot), ((k / kUSlots) & 1) ^ 1);
      if (lane == 0) {
        const Unit U = make_unit(p, unit_index(p, it));
        volatile int32_t* e = uring + 8 * slot;
        e[0] = U.bi;
        e[1] = U.h;
        e[2] = (int32_t)U.row0;
        e[3] = U.n_sink;
        e[4] = U.loc_begin;
        e[5] = U.n_tiles;
        mbar_arrive_local(bar(kBarUFull + slot));
      }
      __syncwarp();
    }
  }
  } else if (warp >= kEpiWarp0) {
    // ===================================================== epilogue warpgroup (warps 12..15, both CTAs)
    // Row r = 32 (warp % 4) + lane, all 128 dims: waits for the unit's row sums (LFull) and last PV (OLast),
    // reads O from TMEM and releases it, stages bf16 [128 x 64] boxes in the unit's dead Q buffer and
    // TMA-stores them; off the softmax warps' path entirely.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    const uint32_t wq = warp & 3, r = wq * 32 + lane;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const uint32_t ofree0 = mapa(bar(kBarOFree), 0);
    const float* lsm = reinterpret_cast<const float*>(smem + kOffLs);
    const float ln2 = 0.69314718055994531f;
    uint32_t uc = 0, g = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = get_unit(uc);
      const uint32_t ob = uc & 1, par = (uc >> 1) & 1;
      g += U.n_tiles;
      mbar_wait(bar(kBarLFull + ob), par);
      const float ltot = lsm[(2 * ob) * 128 + r] + lsm[(2 * ob + 1) * 128 + r];
      const float mrow = lsm[512 + ob * 128 + r];
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarLFree + ob));
      const float inv = 1.0f / ltot;
      mbar_wait(bar(kBarOLast + ob), par);
      tc_fence_after();
      const int64_t row_g = U.row0 + 128 * rank + r;
      const bool row_ok = row_g < p.n_q;
      const uint32_t stage = sbase + kOffQ + kQBytes * ob;  // the unit's Q buffer (its last S has completed)
      float* dst = reinterpret_cast<float*>(p.o) + (int64_t)U.bi * p.o_sb + row_g * p.o_st + (int64_t)U.h * p.o_sh;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        tmem_ld32(taddr + kTmemO + 128 * ob + 32 * c, ov);
        tmem_wait_ld();
        if (p.out_bf16) {
          const uint32_t box = stage + (c >> 1) * kQChunkBytes + r * 128;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(box + ((((c & 1) * 4 + q) ^ (r & 7)) << 4),
                         pack_bf16x2(__uint_as_float(ov[8 * q]) * inv, __uint_as_float(ov[8 * q + 1]) * inv),
                         pack_bf16x2(__uint_as_float(ov[8 * q + 2]) * inv, __uint_as_float(ov[8 * q + 3]) * inv),
                         pack_bf16x2(__uint_as_float(ov[8 * q + 4]) * inv, __uint_as_float(ov[8 * q + 5]) * inv),
                         pack_bf16x2(__uint_as_float(ov[8 * q + 6]) * inv, __uint_as_float(ov[8 * q + 7]) * inv));
        } else if (row_ok) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            st_global_v4(dst + 32 * c + 4 * q, __float_as_uint(__uint_as_float(ov[4 * q]) * inv),
                         __float_as_uint(__uint_as_float(ov[4 * q + 1]) * inv),
                         __float_as_uint(__uint_as_float(ov[4 * q + 2]) * inv),
                         __float_as_uint(__uint_as_float(ov[4 * q + 3]) * inv));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ofree0 + 8 * ob);
      if (warp == kEpiWarp0) MTRACE(9, g - 1);
      if (p.out_bf16) {
        fence_proxy_async_smem();
        named_bar_sync(7, 128);
        if (warp == kEpiWarp0 && lane == 0) {
          for (int m = 0; m < 2; ++m)
            tma_store_5d(&p.o_map, stage + m * kQChunkBytes, 0, (int32_t)(U.row0 + 128 * rank), m, U.h, U.bi);
          bulk_commit_group();
          bulk_wait_group_read0();  // then the Q buffer may be reloaded (unit uc + 2)
          mbar_arrive_local(bar(kBarStageFree + ob));
        }
      } else {
        named_bar_sync(7, 128);
        if (warp == kEpiWarp0 && lane == 0) mbar_arrive_local(bar(kBarStageFree + ob));
      }
      if (p.lse && row_ok) p.lse[((int64_t)U.bi * p.heads + U.h) * p.n_q + row_g] = (mrow + __log2f(ltot)) * ln2;
    }
    if (warp == kEpiWarp0 && lane == 0) bulk_wait_group0();
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 176;");
    // ===================================================== softmax (warps 4..11, both CTAs)
    // lane tl = 32 wq + lane holds row tl; warps with ch take keys / O dims [64 ch, 64 ch + 64). The two warps
    // of a row (wq, ch = 0 / 1) exchange row maxima through smem under named barrier 1 + wq (64 threads).
    // At a unit's end the row's partial sums and max go to the epilogue warpgroup (O is double-buffered in
    // TMEM, so the next unit's tiles proceed while it drains).
    const uint32_t wq = warp & 3;
    const uint32_t ch = (warp - kSmWarp0) >> 2;
    const uint32_t r = wq * 32 + lane;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const uint32_t pfull = mapa(bar(kBarPFull), 0);
    const float sl2 = p.scale_log2;
    const int causal = p.causal, sparse = p.sparse;
    const int64_t n_kv = p.n_kv, sink_keys = (int64_t)p.s * p.b;
    const uint32_t pair_bar = 1 + wq;
    float* lsm = reinterpret_cast<float*>(smem + kOffLs);
    uint32_t g = 0, uc = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = get_unit(uc);
      const int64_t row_g = U.row0 + 128 * rank + r;  // local query token
      const int64_t my_tok = p.q_start + (row_g < p.n_q ? row_g : p.n_q - 1);
      const uint32_t ob = uc & 1;
      int64_t win_lo = 0;  // first local key of this row's window (Eq. 4)
      if (sparse) {
        win_lo = (int64_t)p.div_b.div((uint32_t)my_tok) - p.l + 1;
        if (win_lo < p.s) win_lo = p.s;
        win_lo *= p.b;
      }
      float m_used = -INFINITY, lrow = 0.f;
      for (int i = 0; i < U.n_tiles; ++i, ++g) {
        const uint32_t buf = g & 1;
        const int64_t c0 = sub_k0(U, i) + 64 * ch;
        int64_t lim = n_kv - c0;
        if (causal && my_tok + 1 - c0 < lim) lim = my_tok + 1 - c0;
        if (c0 >= sink_keys && c0 < win_lo) lim = 0;
        const int32_t nvalid = lim < 0 ? 0 : (lim > 64 ? 64 : (int32_t)lim);
        mbar_wait(bar(kBarSFull + buf), (g >> 1) & 1);
        tc_fence_after();
        if (warp == kSmWarp0) MTRACE(6, g);
        const uint32_t sa = taddr + kTmemS + 128 * buf + 64 * ch;
        uint32_t v[64];
        tmem_ld32(sa, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_wait_ld();
        if (nvalid < 64) {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j >= nvalid) v[j] = __float_as_uint(-INFINITY);
        }
        float mx[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // 4 chains of 3-input max over v[4 k + c]
          mx[c] = fmax3(__uint_as_float(v[c]), __uint_as_float(v[4 + c]), __uint_as_float(v[8 + c]));
#pragma unroll
          for (int k = 3; k < 15; k += 2)
            mx[c] = fmax3(mx[c], __uint_as_float(v[4 * k + c]), __uint_as_float(v[4 * k + 4 + c]));
          mx[c] = fmaxf(mx[c], __uint_as_float(v[60 + c]));
        }
        float tmax = fmaxf(fmax3(mx[0], mx[1], mx[2]), mx[3]) * sl2;
        float* rb = red + buf * 256;
        rb[ch * 128 + r] = tmax;
        named_bar_sync(pair_bar, 64);
        tmax = fmaxf(tmax, rb[(ch ^ 1) * 128 + r]);
        const bool resc = tmax > m_used + 8.0f;
        const float m_new = resc ? tmax : m_used;
        const float corr = resc ? ex2(m_used - m_new) : 1.0f;
        const float m_sub = m_new == -INFINITY ? 0.f : m_new;  // a row with no key yet (s = 0, later block)
        // p = 2^(s * scale_log2 - m) on pairs (FFMA2); pairs in kPolyPairs on the FMA pipe, the rest on MUFU
        const uint64_t sl2v = f2pack(sl2, sl2), nmv = f2pack(-m_sub, -m_sub);
        uint64_t acc0 = f2pack(0.f, 0.f), acc1 = acc0;
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint64_t y = ffma2(f2pack(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), sl2v, nmv);
          uint64_t e;
          if ((kPolyPairs >> j) & 1u) {
            e = exp2_poly2(y);
          } else {
            float y0, y1;
            f2unpack(y, y0, y1);
            e = f2pack(ex2(y0), ex2(y1));
          }
          if (j & 1)
            acc1 = fadd2(acc1, e);
          else
            acc0 = fadd2(acc0, e);
          float e0, e1;
          f2unpack(e, e0, e1);
          pk[j] = pack_bf16x2(e0, e1);
        }
        float ps0, ps1;
        f2unpack(fadd2(acc0, acc1), ps0, ps1);
        if (i > 0 && __any_sync(0xffffffffu, resc)) {  // rescale O once PV(g - 1) has landed
          const uint32_t gp = g - 1;
          mbar_wait(bar(kBarOFull + (gp & 1)), (gp >> 1) & 1);
          tc_fence_after();
          if (warp == kSmWarp0) MTRACE(7, g);
          {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint32_t ov[32];
              tmem_ld32(taddr + kTmemO + 128 * ob + 64 * ch + 32 * hh, ov);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
              tmem_st32(taddr + kTmemO + 128 * ob + 64 * ch + 32 * hh, ov);
            }
            tmem_wait_st();
          }
        }
        // P (bf16) over this thread's S columns: keys 64 ch .. 64 ch + 63 -> cols 32 ch .. 32 ch + 31. The pair
        // barrier above ordered both threads' S loads before either P store.
        tmem_st32(taddr + kTmemS + 128 * buf + 32 * ch, pk);
        lrow = lrow * corr + (ps0 + ps1);
        m_used = m_new;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(pfull);
        if (warp == kSmWarp0) MTRACE(8, g);
      }
      // the unit's row sums / max to the epilogue warpgroup (after it has read unit uc - 2's)
      mbar_wait(bar(kBarLFree + ob), ((uc >> 1) & 1) ^ 1);
      lsm[(2 * ob + ch) * 128 + r] = lrow;
      if (ch == 0) lsm[512 + ob * 128 + r] = m_used;
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarLFull + ob));
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

extern unsigned long long* g_debug_trace;  // attn_tc_prefill.cu (loza_debug_set_trace)

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
  p.trace = g_debug_trace;
  const int64_t upb = (a.n_q + 255) / 256, total = upb * a.batch * a.heads;
  if (total >= ((int64_t)1 << 31)) return cudaErrorInvalidValue;
  p.units_per_bh = (uint32_t)upb;
  p.total_units = (uint32_t)total;
  p.div_upb.init((uint32_t)upb);
  p.div_heads.init((uint32_t)a.heads);
  p.div_b.init((uint32_t)p.b);
  if (p.total_units == 0) return cudaSuccess;
  const KvSeg& s = a.kv.seg[0];
  const uint64_t H = (uint64_t)a.heads;
  if (!encode_5d_heads(&p.q_map, a.q, kDqk, (uint64_t)a.n_q, H, a.batch, a.q_st, a.q_sh, a.q_sb, 128, 1) ||
      !encode_5d_heads(&p.k_map, s.k, kDqk, (uint64_t)a.n_kv, H, a.batch, s.k_st, k_sh, s.k_sb, 64, 3) ||
      !encode_5d_heads(&p.v_map, s.v, kDv, (uint64_t)a.n_kv, H, a.batch, s.v_st, v_sh, s.v_sb, 128, 1))
    return cudaErrorInvalidValue;
  if (a.out_bf16 && !encode_5d_heads(&p.o_map, a.o, kDv, (uint64_t)a.n_q, H, a.batch, a.o_st, a.o_sh, a.o_sb, 128, 1))
    return cudaErrorInvalidValue;
  {  // per launch (the attribute is per device; a process may drive several GPUs)
    cudaError_t e = cudaFuncSetAttribute(prefill_mha_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  int64_t ncl = sms / 2;
  if (ncl > p.total_units) ncl = p.total_units;
  prefill_mha_kernel<<<(unsigned)(2 * ncl), kThreads, kSmemAlloc, st>>>(p);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza
