// SSA decode, pair-cooperative (Eq. 4 at p = seq_len - 1): the two CTAs of a cluster work on
// the SAME 256-key tiles with cta_group::2 UMMAs, so the window needs no cross-CTA merge at the end.
//
//  * A pair tile = two selected 128-key sub-blocks; CTA r stages sub-block 2i + r (its 128 keys) and half of Q
//    (heads 32 r .. 32 r + 31). S^T = K Q^T: 36 UMMAs M256 (keys: 128 per CTA) N64 (heads; B split 32/32)
//    K16 -> each CTA's TMEM holds S^T of its own 128 keys x all 64 heads. One UMMA stream feeds both SMs
//    (M256 N64: 43 cycles for the pair vs 2 x 48 for two M128 N64 streams).
//  * Softmax per CTA over its own keys with a SHARED running max per head: each CTA reduces its per-head tile
//    maximum and swaps the 64 values with the partner through DSMEM, so both CTAs use the same max and
//    their P values can enter one MMA; lane j of a warp takes the lazy-rescale decision for head j and the
//    warp reads the 32 (m, corr) pairs back as smem broadcasts. A thread (key k, heads 32 ch ..) writes its
//    32 P values (64 B): own heads into this CTA's P half, the partner's heads into a staging block that the
//    transfer warp moves with ONE 8 KB bulk DSMEM copy (completion on the receiver's barrier, spin-waited);
//    P_r = [256 keys][32 heads] bf16, SWIZZLE_64B MN-major (the B operand half of CTA r).
//  * O^T += V^T P: 32 UMMAs M256 (dims: CTA r owns dims [256 r, 256 r + 256), two 128-dim groups) N64
//    (heads) K16 over all 256 keys; each CTA streams V rows of both sub-blocks for its 256 dims. The per-head
//    sums l are swapped once at the end through an mbarrier (the other roles do not wait); each CTA
//    normalises its own dims and stores them straight from registers (lane pairs swap one value per head pair
//    so every store is a bf16x2); the final cluster barrier is relaxed (no wait for the stores to drain).
//  * S runs two tiles ahead of PV (MMA order S(0), S(1), S(2), PV(0), S(3), PV(1), ..., three S^T buffers in
//    TMEM) so the HBM-bound K rows of tile i + 2 are in flight while P(i) is being made; the softmax of tile i
//    waits for PV(i - 2) before it rewrites that tile's P buffer and staging block.
//  * H < 64 (a head-sharded GPU): the Q rows >= H are TMA zero-fill (the padded heads' columns are computed and
//    dropped at the store); the work is that of H = 64, which is still faster than the key-split kernel
//    (attn_tc_decode_ks.cu, now reachable through the test knob only): the window's bytes dominate.
//  * Up to 10 helper clusters on the SMs the pairs leave idle L2-prefetch the later pair tiles' cache rows (paced
//    by the global timer), so the pairs' TMA loads of those tiles mostly hit L2.
//  * Loads: warp 0 of each CTA (Q halves first through 9 chunk barriers; then a ring of 4 x 32 KB items in
//    MMA order K(0), K(1), K(2), V(0), K(3), V(1), ...; pair TMA with completion on the leader's barriers);
//    warp 1 of the leader issues every UMMA; warps 2-9 of both CTAs run the softmax.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

#ifndef DECODE_EARLY_PF
#define DECODE_EARLY_PF 1
#endif
// Helper clusters on the SMs the pairs leave idle (B < SMs / 2): they L2-prefetch every sequence's cache rows of
// pair tiles 1, 2, ... (tile t issued (t - 1) x kHelperDelta ns after the dependency wait). Measured (B64 at 128K,
// bench timing, one box): no helpers 22.4 us; 10 helper clusters 21.2 us for any pacing 0-3.5 us; the same
// clusters idle 22.85; prefetching tile 1 only 23.1, tiles 2.. only 23.5, tiles 0.. 23.4; 5 clusters 29.5.
#ifndef DECODE_HELPER_CLUSTERS
#define DECODE_HELPER_CLUSTERS 10
#endif
constexpr int kHelperClusters = DECODE_HELPER_CLUSTERS;
constexpr unsigned long long kHelperDelta = 2000;

namespace loza {

namespace {
using namespace sm100;

constexpr int kDqk = 576, kDv = 512, kChunks = 9, kH = 64;
constexpr int kThreads = 352;  // warp 0 TMA, warp 1 MMA (leader), warps 2-9 softmax / epilogue, warp 10 P transfer
constexpr int kXferWarp = 10;
constexpr int kStageBytes = 32768, kHalf = 16384;
constexpr int kStages = 4;
constexpr int kQChunk = 32 * 128;                // 32 heads x 64 dims
constexpr int kQBytes = kChunks * kQChunk;       // 36864
constexpr int kPBytes = 256 * 64;                // [256 keys][32 heads] bf16 per buffer
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;           // 2 buffers
constexpr int kOffPst = kOffP + 2 * kPBytes;     // staging of the partner's P rows [2 buf][128 keys][32 heads]
constexpr int kPstBytes = 128 * 64;
constexpr int kOffRing = kOffPst + 2 * kPstBytes;
constexpr int kOffBar = kOffRing + kStages * kStageBytes;
constexpr int kBarFull = 0;
constexpr int kBarEmpty = kBarFull + kStages;
constexpr int kBarQFull = kBarEmpty + kStages;    // [9]
// S runs kAhead tiles ahead of PV. Measured (B64 at 128K, bench timing): 1 (FA order) 22.2 us, 2 21.1-21.2,
// 3 21.85, 4 21.98 -- beyond 2 the V re-reads bunch up behind the last K tile
constexpr int kAhead = 2;  // with the helper clusters: 1 21.8 us, 2 21.3, 3 22.4
constexpr int kSBufs = kAhead + 1;                // S^T buffers in TMEM
constexpr int kBarSFull = kBarQFull + kChunks;    // [kSBufs]
constexpr int kBarSFree = kBarSFull + kSBufs;     // [kSBufs]
constexpr int kBarPFull = kBarSFree + kSBufs;     // [2]
constexpr int kBarOFull = kBarPFull + 2;          // [2]
constexpr int kBarMax = kBarOFull + 2;            // [2] partner's tile maxima landed (bulk copy, local)
constexpr int kBarPStaged = kBarMax + 2;          // [2] the partner's-heads P rows are staged (4 warps, local)
constexpr int kBarPRecv = kBarPStaged + 2;         // [2] the partner's P rows landed here (bulk copy, local)
constexpr int kBarL = kBarPRecv + 2;              // partner's sums landed (local)
constexpr int kNumBars = kBarL + 1;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffRed = (kOffTmemPtr + 4 + 15) & ~15;  // float [2 buf][4 key quarters][64 heads]
constexpr int kOffX = kOffRed + 2 * 4 * 64 * 4;       // float partner maxima [2 buf][64], partner sums [64]
constexpr int kOffXl = kOffX + 3 * 64 * 4;            // float own maxima [2 buf][64], own sums [64] (copy sources)
constexpr int kOffInv = kOffXl + 3 * 64 * 4;          // float 1/l [64]
constexpr int kOffHm = kOffInv + 64 * 4;             // float per softmax warp: -m [32], corr [32]
constexpr int kSmemUsed = kOffHm + 8 * 64 * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 0, kTmemS = 128;  // O^T group g at 64 g (lanes = dims), S^T buffer b at 128 + 64 b
constexpr uint32_t kSoftmaxWarps = 8;
constexpr uint32_t kSmThreads = 32 * kSoftmaxWarps;
constexpr uint32_t kArrivalsPerPair = 2 * kSoftmaxWarps;
constexpr uint32_t kPFullArrivals = kArrivalsPerPair + 2;  // + the transfer warp of each CTA

struct CoopParams {
  CUtensorMap q_map, k_map, v_map;
  const int32_t* seq_lens;
  int32_t batch, heads, s, l, b;  // heads <= 64: a head-sharded GPU's Q rows >= heads are TMA zero-fill
  int32_t ring;
  int64_t t_cap;
  int32_t n_rows;  // cache rows (an absent sub-block maps here: out of bounds, zero-filled)
  const uint8_t* kraw;  // contiguous cache rows (L2 prefetch before the dependency wait), or NULL
  const uint8_t* qraw;  // contiguous Q rows, or NULL
  int64_t k_sb_bytes, k_st_bytes, q_sb_bytes;
  float scale_log2;
  void* o;
  int64_t o_sb, o_sh;
  int32_t out_bf16;
  float* lse;
  unsigned long long* trace;  // debug timeline of cluster trace_cluster (NULL in production): [slot][rank][16]
  int32_t trace_cluster;
  int32_t* status;  // nullable: LOZA_ERR_SHAPE when a seq_len was outside [1, t_cap] (clamped)
};

#define CTRACE(slot, idx)                                                                         \
  do {                                                                                            \
    if (p.trace && (int)(blockIdx.x >> 1) == p.trace_cluster && (idx) < 16 && (threadIdx.x & 31) == 0) \
      p.trace[((slot) * 2 + cluster_ctarank()) * 16 + (idx)] = clock64();                       \
  } while (0)

// S^T buffer of tile gi and the parity of its use
__device__ __forceinline__ uint32_t sbuf(uint32_t gi) { return gi % kSBufs; }
__device__ __forceinline__ uint32_t sphase(uint32_t gi) { return (gi / kSBufs) & 1; }
struct SeqTiles {
  int32_t n_sink, loc_begin, n_tiles;  // selected 128-key sub-blocks
  int32_t pos;
};
__device__ __forceinline__ SeqTiles seq_tiles(const CoopParams& p, int bi) {
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
// absolute first key of selected sub-block j, or -1 past the list
__device__ __forceinline__ int32_t sub_k0(const SeqTiles& t, int j) {
  if (j >= t.n_tiles) return -1;
  return (j < t.n_sink ? j : t.loc_begin + (j - t.n_sink)) * 128;
}
// cache row of key k0: identity, or the ring slot of its block; an absent sub-block -> n_rows (OOB)
__device__ __forceinline__ int32_t kv_row(const CoopParams& p, int32_t k0) {
  if (k0 < 0) return p.n_rows;
  if (!p.ring) return k0;
  const int32_t kb = k0 / p.b;
  if (kb < p.s) return k0;
  return p.s * p.b + ((kb - p.s) % p.l) * p.b + (k0 - kb * p.b);
}
// smem descriptor, SWIZZLE_64B (layout type 4), version 1
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
__device__ __forceinline__ void st_shared_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

#define FULL_L(slot) (full_l + 8 * (slot))
#define GSTAMP(k)                                                       \
  do {                                                                  \
    if (p.trace && threadIdx.x == 64) {                                 \
      unsigned long long g_;                                            \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_));             \
      p.trace[11 * 2 * 16 + 8 * blockIdx.x + (k)] = g_;                 \
    }                                                                   \
  } while (0)

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    decode_coop_kernel(const __grid_constant__ CoopParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  float* xch = reinterpret_cast<float*>(smem + kOffX);
  float* invl = reinterpret_cast<float*>(smem + kOffInv);
  const uint32_t rank = cluster_ctarank(), partner = rank ^ 1;
  const int bi = (int)(blockIdx.x >> 1);
  if (bi >= p.batch) {  // helper cluster (idle SMs): L2 prefetch of the sequences' later pair tiles, paced
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x >= 32 || !p.kraw) return;
    const int hid = (int)blockIdx.x - 2 * p.batch, nh = (int)gridDim.x - 2 * p.batch;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int t = 1;; ++t) {
      {
        unsigned long long g;
        do {
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        } while (g < t0 + (unsigned long long)(t - 1) * kHelperDelta);
      }
      bool any = false;
      for (int sq = hid; sq < p.batch; sq += nh) {
        const SeqTiles sqt = seq_tiles(p, sq);
        if (2 * t >= sqt.n_tiles) continue;
        any = true;
        if (lane < 2) {
          const int32_t k0 = sub_k0(sqt, 2 * t + (int)lane);
          if (k0 >= 0) {
            const int32_t row = kv_row(p, k0);
            int32_t nr = p.n_rows - row;
            nr = nr > 128 ? 128 : nr;
            if (nr > 0) bulk_prefetch_l2(p.kraw + sq * p.k_sb_bytes + row * p.k_st_bytes, (uint32_t)(nr * p.k_st_bytes));
          }
        }
      }
      if (!__any_sync(0xffffffffu, any)) break;
    }
    return;
  }

  if (p.trace && threadIdx.x == 0) {  // per-CTA wall-clock span (globaltimer ns) after the timeline slots
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[11 * 2 * 16 + 8 * blockIdx.x] = g;
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar(kBarFull + i), 1);
      mbar_init(bar(kBarEmpty + i), 1);
    }
    for (int i = 0; i < kChunks; ++i) mbar_init(bar(kBarQFull + i), 1);
    for (int i = 0; i < kSBufs; ++i) {
      mbar_init(bar(kBarSFull + i), 1);
      mbar_init(bar(kBarSFree + i), kArrivalsPerPair);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarPFull + i), kPFullArrivals);
      mbar_init(bar(kBarOFull + i), 1);
      mbar_init(bar(kBarMax + i), 1);    // armed each tile (expect_tx 256 B), completed by the partner's copies
      mbar_init(bar(kBarPStaged + i), 4);
      mbar_init(bar(kBarPRecv + i), 1);  // armed each tile (expect_tx 8 KB), completed by the partner's copy
    }
    mbar_init(bar(kBarL), 2);  // the partner's two writer warps
    fence_mbar_init();
    // every barrier a partner's bulk copy completes is armed BEFORE that copy can arrive (here for the first
    // phases, then one phase ahead by the thread that consumed the previous one): a complete_tx that reaches
    // an unarmed barrier was measured to stall the copy by ~20 us
    for (int i = 0; i < 2; ++i) {
      mbar_arrive_expect_tx(bar(kBarMax + i), 64 * 4);
      mbar_arrive_expect_tx(bar(kBarPRecv + i), kPstBytes);
    }
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.k_map);
    prefetch_tmap(&p.v_map);
  }
  if (warp == 1) tmem_alloc<2>(smem_u32(tmem_ptr_smem), kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;
#if DECODE_EARLY_PF
  // Under programmatic dependent launch this CTA may start while the previous kernel still runs. Before
  // waiting for it, pull the first pair tile's cache rows (both sub-blocks: this CTA's K, and V for its
  // dims) and this CTA's Q half into L2: hints only (seq_lens read here may be stale; nothing is consumed
  // before the wait), so the first loads after the wait hit L2 instead of paying the HBM latency.
  if (warp == 0 && lane == 0 && p.kraw) {
    const SeqTiles s0 = seq_tiles(p, bi);
    for (int j = 0; j < 2; ++j) {
      const int32_t k0 = sub_k0(s0, j);
      if (k0 < 0) continue;
      const int32_t row = kv_row(p, k0);
      int32_t nr = p.n_rows - row;
      nr = nr > 128 ? 128 : nr;
      if (nr > 0) bulk_prefetch_l2(p.kraw + bi * p.k_sb_bytes + row * p.k_st_bytes, (uint32_t)(nr * p.k_st_bytes));
    }
    const int nh = p.heads - 32 * (int)rank;  // this CTA's real Q rows
    if (p.qraw && nh > 0)
      bulk_prefetch_l2(p.qraw + bi * p.q_sb_bytes + rank * 32 * kDqk * 2, (uint32_t)((nh < 32 ? nh : 32) * kDqk * 2));
  }
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");  // inputs of the previous kernel are visible from here
  if (p.trace && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[11 * 2 * 16 + 8 * blockIdx.x + 1] = g;
  }

  const SeqTiles st = seq_tiles(p, bi);
  const int npt = (st.n_tiles + 1) / 2;  // pair tiles (>= 1)
  if (p.status && threadIdx.x == 0 && cluster_ctarank() == 0) {
    const int64_t L = p.seq_lens[bi];
    if (L < 1 || L > p.t_cap) atomicExch(p.status, (int32_t)LOZA_ERR_SHAPE);
  }
  CTRACE(0, 0);

  if (warp == 0) {
    // ----------------------------------------------------- TMA producer (each CTA: its Q half, keys, V dims)
    const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
    const uint32_t full_l = mapa(bar(kBarFull), 0), qfull_l = mapa(bar(kBarQFull), 0);
    for (int c = 0; c < kChunks; ++c) {
      if (elect_one()) {
        if (rank == 0) mbar_arrive_expect_tx(bar(kBarQFull + c), 2 * kQChunk);
        tma_load_3d_pair(sbase + kOffQ + c * kQChunk, &p.q_map, 64 * c, 32 * (int)rank, bi, qfull_l + 8 * c, pol_q);
      }
      __syncwarp();
    }
    uint32_t slot = 0, phase = 0;
    auto acquire = [&]() -> uint32_t {
      mbar_wait(bar(kBarEmpty + slot), phase ^ 1);
      return sbase + kOffRing + slot * kStageBytes;
    };
    auto next = [&]() {
      if (++slot == kStages) {
        slot = 0;
        phase ^= 1;
      }
    };
    auto load_k = [&](int i) {  // this CTA's sub-block of pair tile i: 5 items of 2 chunks (chunk 8 alone)
      const int32_t row = kv_row(p, sub_k0(st, 2 * i + (int)rank));
      for (int j = 0; j < (kChunks + 1) / 2; ++j) {
        const uint32_t dst = acquire();
        const int nc = 2 * j + 1 < kChunks ? 2 : 1;
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + slot), 2 * nc * kHalf);
          for (int sub = 0; sub < nc; ++sub)
            tma_load_3d_pair(dst + kHalf * sub, &p.k_map, 64 * (2 * j + sub), row, bi, FULL_L(slot), pol_kv);
        }
        __syncwarp();
        next();
      }
    };
    auto load_v = [&](int i) {  // pair tile i's 256 keys x this CTA's 256 dims: 4 items of 64 keys
      for (int q = 0; q < 4; ++q) {
        const int32_t k0 = sub_k0(st, 2 * i + (q >> 1));
        const int32_t row = k0 < 0 ? p.n_rows : kv_row(p, k0) + 64 * (q & 1);
        const uint32_t dst = acquire();
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + slot), 2 * kStageBytes);
          for (int sub = 0; sub < 2; ++sub)  // 32 keys x dim chunks 4 r .. 4 r + 3 ([chunk][32 keys][64 dims])
            tma_load_4d_pair(dst + kHalf * sub, &p.v_map, 0, row + 32 * sub, 4 * (int)rank, bi, FULL_L(slot), pol_kv);
        }
        __syncwarp();
        next();
      }
    };
    for (int i = 0; i < kAhead && i < npt; ++i) load_k(i);
    for (int i = 0; i < npt; ++i) {
      if (i + kAhead < npt) load_k(i + kAhead);
      load_v(i);
    }
  } else if (warp == 1) {
    // ----------------------------------------------------- UMMA issuer (leader CTA)
    if (rank == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(256, 64, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(256, 64, true, true);
      const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
      const uint64_t dk = sdesc_sw128(sbase + kOffRing, 16, 1024);
      const uint64_t dv = sdesc_sw128(sbase + kOffRing, 4096, 1024);  // V^T: [chunk][keys][64 dims], MN-major
      const uint64_t dp = sdesc_sw64(sbase + kOffP, 16, 512);         // P_r: [keys][32 heads], MN-major
      uint32_t slot = 0, phase = 0;
      auto next = [&]() {
        if (++slot == kStages) {
          slot = 0;
          phase ^= 1;
        }
      };
      auto issue_s = [&](uint32_t gi) {
        const uint32_t buf = sbuf(gi);
        CTRACE(1, gi);
        mbar_wait(bar(kBarSFree + buf), sphase(gi) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + kTmemS + 64 * buf;
        for (int j = 0; j < (kChunks + 1) / 2; ++j) {
          const int nc = 2 * j + 1 < kChunks ? 2 : 1;
          if (gi == 0)
            for (int sub = 0; sub < nc; ++sub) mbar_wait(bar(kBarQFull + 2 * j + sub), 0);
          mbar_wait(bar(kBarFull + slot), phase);
          tc_fence_after();
          if (elect_one()) {
            for (int sub = 0; sub < nc; ++sub) {
              const int cc = 2 * j + sub;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                umma_bf16_pair(d, dk + (uint64_t)((kStageBytes * slot + kHalf * sub + 32 * k) >> 4),
                               dq + (uint64_t)((kQChunk * cc + 32 * k) >> 4), idesc_s, (cc | k) != 0);
            }
            umma_commit_pair_mc(bar(kBarEmpty + slot), 3);
          }
          __syncwarp();
          next();
        }
        if (elect_one()) umma_commit_pair_mc(bar(kBarSFull + buf), 3);
        __syncwarp();
        CTRACE(2, gi);
      };
      auto issue_pv = [&](uint32_t gi, bool first) {
        const uint32_t buf = gi & 1;
        CTRACE(3, gi);
        mbar_wait_acquire_cluster(bar(kBarPFull + buf), (gi >> 1) & 1);

        CTRACE(4, gi);  // the partner's DSMEM writes of this P half are visible before the MMA reads it
        tc_fence_after();
        for (int q = 0; q < 4; ++q) {
          mbar_wait(bar(kBarFull + slot), phase);
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int sub = 0; sub < 2; ++sub)
#pragma unroll
              for (int kk = 0; kk < 2; ++kk)
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                  const int key = 64 * q + 32 * sub + 16 * kk;  // of the 256-key pair tile
                  umma_bf16_pair(tmem + kTmemO + 64 * g,
                                 dv + (uint64_t)((kStageBytes * slot + kHalf * sub + 8192 * g + 2048 * kk) >> 4),
                                 dp + (uint64_t)((kPBytes * buf + key * 64) >> 4), idesc_pv,
                                 !(first && key == 0));
                }
            umma_commit_pair_mc(bar(kBarEmpty + slot), 3);
          }
          __syncwarp();
          next();
        }
        if (elect_one()) umma_commit_pair_mc(bar(kBarOFull + buf), 3);
        __syncwarp();
        CTRACE(5, gi);
      };
      for (int i = 0; i < kAhead && i < npt; ++i) issue_s((uint32_t)i);
      for (int i = 0; i < npt; ++i) {
        if (i + kAhead < npt) issue_s((uint32_t)(i + kAhead));
        issue_pv((uint32_t)i, i == 0);
      }
      // the last tiles' S-buffer releases (remote arrivals from the partner) land before this CTA can exit:
      // the final cluster barrier is relaxed
      for (int j = npt - kSBufs; j < npt; ++j)
        if (j >= 0) mbar_wait(bar(kBarSFree + sbuf((uint32_t)j)), sphase((uint32_t)j));
    }
  } else if (warp == kXferWarp) {
    // ----------------------------------------------------- P transfer (each CTA): the staged rows of the
    // partner's heads (8 KB) into rows 128 rank .. of the partner's P half, off the softmax warps' path
    const uint32_t pfull0 = mapa(bar(kBarPFull), 0);
    for (int i = 0; i < npt; ++i) {
      const uint32_t buf = (uint32_t)i & 1, ph = ((uint32_t)i >> 1) & 1;
      mbar_wait(bar(kBarPStaged + buf), ph);
      if (lane == 0)
        bulk_copy_to_cluster(mapa(sbase + kOffP + buf * kPBytes + 128 * rank * 64, partner),
                             sbase + kOffPst + buf * kPstBytes, kPstBytes, mapa(bar(kBarPRecv + buf), partner));
      mbar_wait_spin(bar(kBarPRecv + buf), ph);  // the partner's rows of this CTA's P half landed
      if (lane == 0) {
        if (i + 2 < npt) mbar_arrive_expect_tx(bar(kBarPRecv + buf), kPstBytes);  // tile i + 2, armed ahead
        mbar_arrive_release_cluster(pfull0 + 8 * buf);
      }
      __syncwarp();
    }
  } else {
    // ----------------------------------------------------- softmax (warps 2..9 of both CTAs)
    // TMEM lane quarter wq = warp % 4: S^T lanes = this CTA's keys 32 wq .. 32 wq + 31 of its sub-block; column
    // half ch selects heads [32 ch, 32 ch + 32). Per-head tile maxima: redux.sync over the warp's keys, the 4
    // key-quarter warps through smem, then the partner's via DSMEM (the warps with wq == 0 send).
    const uint32_t wq = warp & 3;
    const uint32_t ch = (warp - 2) >> 2;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const uint32_t kl = 32 * wq + lane;           // key within this CTA's sub-block
    const uint32_t prow = 128 * rank + kl;        // row in the 256-key pair tile
    const float sl2 = p.scale_log2;
    const uint32_t sfree0 = mapa(bar(kBarSFree), 0), pfull0 = mapa(bar(kBarPFull), 0);
    float m_used[32], lpart[32];
    float m_mine = -INFINITY;  // lane j: running max of head 32 ch + j
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      m_used[j] = -INFINITY;
      lpart[j] = 0.f;
    }
    for (int i = 0; i < npt; ++i) {
      const uint32_t gi = (uint32_t)i, buf = gi & 1, sb = sbuf(gi);
      const int32_t kb0 = sub_k0(st, 2 * i + (int)rank);
      const bool kvalid = kb0 >= 0 && kb0 + (int32_t)kl <= st.pos;
      mbar_wait(bar(kBarSFull + sb), sphase(gi));
      if (warp == 2) CTRACE(6, gi);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(taddr + kTmemS + 64 * sb + 32 * ch, v);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(sfree0 + 8 * sb);
      float* rb = red + buf * 256;
      float wmax_mine = -INFINITY;  // lane j keeps head 32 ch + j
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (!kvalid) v[j] = __float_as_uint(-INFINITY);
        const float x = __uint_as_float(v[j]);
        float r;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
        if (j == (int)lane) wmax_mine = r;
      }
      rb[wq * 64 + 32 * ch + lane] = wmax_mine;
      named_bar_sync(1, kSmThreads);
      const float cmax = fmaxf(fmaxf(rb[32 * ch + lane], rb[64 + 32 * ch + lane]),
                               fmaxf(rb[128 + 32 * ch + lane], rb[192 + 32 * ch + lane]));  // this CTA's keys
      if (wq == 0) {  // send this CTA's maxima for heads 32 ch .. to the partner (one 128-B bulk DSMEM copy)
        const uint32_t src = sbase + kOffXl + (buf * 64 + 32 * ch) * 4;
        st_shared_f32(src + lane * 4, cmax);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0)
          bulk_copy_to_cluster(mapa(sbase + kOffX + (buf * 64 + 32 * ch) * 4, partner), src, 128,
                               mapa(bar(kBarMax + buf), partner));
      }
      if (warp == 2) CTRACE(7, gi);
      mbar_wait_spin(bar(kBarMax + buf), (gi >> 1) & 1);
      if (warp == 2 && lane == 0 && i + 2 < npt) mbar_arrive_expect_tx(bar(kBarMax + buf), 64 * 4);  // tile i + 2
      if (warp == 2) CTRACE(8, gi);
      const float hmax = fmaxf(cmax, xch[buf * 64 + 32 * ch + lane]) * sl2;  // shared by both CTAs
      uint32_t pk[16];
      // lane j decides head 32 ch + j (lazy rescale at 2^8); the warp's 32 (-m, corr) pairs are read back as
      // broadcast float4s instead of 32 shuffles + 32 uniform branches per tile
      bool any_resc;
      float corr[32];
      {
        float* hm = reinterpret_cast<float*>(smem + kOffHm) + (warp - 2) * 64;
        const bool resc = hmax > m_mine + 8.0f;
        const float m_new = resc ? hmax : m_mine;
        const float cr = resc ? ex2(m_mine - m_new) : 1.0f;
        m_mine = m_new;
        any_resc = __any_sync(0xffffffffu, resc);
        __syncwarp();  // the previous tile's reads of this slot are done
        hm[lane] = -m_new;
        hm[32 + lane] = cr;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 a = *reinterpret_cast<const float4*>(hm + 4 * q);
          m_used[4 * q] = a.x;
          m_used[4 * q + 1] = a.y;
          m_used[4 * q + 2] = a.z;
          m_used[4 * q + 3] = a.w;
        }
        if (any_resc) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 c = *reinterpret_cast<const float4*>(hm + 32 + 4 * q);
            corr[4 * q] = c.x;
            corr[4 * q + 1] = c.y;
            corr[4 * q + 2] = c.z;
            corr[4 * q + 3] = c.w;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) lpart[j] *= corr[j];
        }
      }
      {
        const uint64_t s2 = f2pack(sl2, sl2);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {  // m_used holds -m here; invalid keys are -inf -> 0
          float x0, x1;
          f2unpack(ffma2(f2pack(__uint_as_float(v[j]), __uint_as_float(v[j + 1])), s2, f2pack(m_used[j], m_used[j + 1])),
                   x0, x1);
          const float e0 = ex2(x0), e1 = ex2(x1);
          lpart[j] += e0;
          lpart[j + 1] += e1;
          pk[j >> 1] = pack_bf16x2(e0, e1);
        }
      }
      // P row of CTA ch's half: 64 B = 4 x 16-B units, SWIZZLE_64B (unit ^ (row >> 1) & 3; rows 128 r + kl
      // and kl share the pattern). Own heads: straight into this CTA's P half; the partner's heads: into the
      // staging block that one bulk DSMEM copy moves to rows 128 rank .. of the partner's half.
      // S(i) completing no longer implies PV(i - 2) completed (S runs two tiles ahead): the P buffer and the
      // staging block of tile i - 2 are free once PV(i - 2) has landed
      if (i >= 2) mbar_wait(bar(kBarOFull + (buf)), ((gi - 2) >> 1) & 1);
      const uint32_t pr = ch == rank ? sbase + kOffP + buf * kPBytes + prow * 64 : sbase + kOffPst + buf * kPstBytes + kl * 64;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        st_shared_v4(pr + ((u ^ ((kl >> 1) & 3)) << 4), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
      if (ch != rank) {  // staged for the transfer warp
        fence_proxy_async_smem();  // the bulk copy (async proxy) reads the staged rows
        __syncwarp();
        if (lane == 0) mbar_arrive_local(bar(kBarPStaged + buf));
      }
      // O^T rescale once PV(i - 1) has landed -- only when a head's max moved
      if (i > 0 && __any_sync(0xffffffffu, any_resc)) {  // corr is per head: uniform across a warp with this ch
        const uint32_t gp = gi - 1;
        mbar_wait(bar(kBarOFull + (gp & 1)), (gp >> 1) & 1);
        tc_fence_after();
        {
#pragma unroll 1
          for (int g = 0; g < 2; ++g) {
            uint32_t ov[32];
            tmem_ld32(taddr + kTmemO + 64 * g + 32 * ch, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr[j]);
            tmem_st32(taddr + kTmemO + 64 * g + 32 * ch, ov);
          }
          tmem_wait_st();
        }
      }
      tc_fence_before();
      if (ch == rank) {
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(pfull0 + 8 * buf);
      } else {  // (its O^T rescale is done; its P rows travel with the transfer warp)
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(pfull0 + 8 * buf);
      }
      if (warp == 2) CTRACE(9, gi);
    }
    if (p.trace && threadIdx.x == 64) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
      p.trace[11 * 2 * 16 + 8 * blockIdx.x + 2] = g;
    }
    if (p.trace && lane == 0) {  // every softmax warp: left the tile loop
      unsigned long long g;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
      p.trace[11 * 2 * 16 + 8 * 2 * p.batch + 8 * blockIdx.x + (warp - 2)] = g;
    }
    // ---------------- l[h] = this CTA's keys' sum + the partner's (mbarrier swap: no wait for the other roles)
    const uint32_t gl = (uint32_t)(npt - 1);
    float lmine;  // lane j: this warp's key-quarter sum for head 32 ch + j (transpose-reduce, 31 shuffles)
    {
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = lpart[j];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & (uint32_t)o) != 0;
#pragma unroll
        for (int k = 0; k < o; ++k) {
          const float send = up ? v[k] : v[k + o];
          const float keep = up ? v[k + o] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      lmine = v[0];
    }
    float* ls = red + ((gl + 1) & 1) * 256;
    ls[wq * 64 + 32 * ch + lane] = lmine;
    named_bar_sync(1, kSmThreads);
    const float lc = (ls[32 * ch + lane] + ls[64 + 32 * ch + lane]) + (ls[128 + 32 * ch + lane] + ls[192 + 32 * ch + lane]);
    if (wq == 0) {
      st_cluster_f32(mapa(sbase + kOffX + (128 + 32 * ch + lane) * 4, partner), lc);
      __syncwarp();
      if (lane == 0) mbar_arrive_release_cluster(mapa(bar(kBarL), partner));
      if (warp == 2) CTRACE(10, 0);
      mbar_wait_acquire_cluster(bar(kBarL), 0);
      const float lt = lc + xch[128 + 32 * ch + lane];
      const uint32_t h = 32 * ch + lane;
      invl[h] = 1.0f / lt;
      const float mh = m_mine;
      if (p.lse && rank == 0 && h < (uint32_t)p.heads)
        p.lse[(int64_t)bi * p.heads + h] = (mh * 0.69314718055994531f) + __logf(lt);
    }
    mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
    if (warp == 2) CTRACE(10, 1);
    tc_fence_after();
    named_bar_sync(1, kSmThreads);  // invl written
    if (warp == 2) CTRACE(10, 3);
    float w[32];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 w4 = *reinterpret_cast<const float4*>(invl + 32 * ch + 4 * q);
      w[4 * q] = w4.x;
      w[4 * q + 1] = w4.y;
      w[4 * q + 2] = w4.z;
      w[4 * q + 3] = w4.w;
    }
    // O^T (lanes = dims 128 g + 32 wq + lane of this CTA's 256, cols = heads) / l -> O[b][h][dim] straight from
    // registers: lanes 2d, 2d + 1 swap one value per head pair so each stores two adjacent dims (bf16x2)
    const uint32_t t = 32 * wq + lane;
    const bool even = (lane & 1) == 0;
    uint32_t ovg[2][32];
    tmem_ld32(taddr + kTmemO + 32 * ch, ovg[0]);
    tmem_ld32(taddr + kTmemO + 64 + 32 * ch, ovg[1]);
    tmem_wait_ld();
    if (warp == 2) CTRACE(10, 6);
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      if (g == 1 && warp == 2) CTRACE(10, 7);
      const uint32_t(&ov)[32] = ovg[g];
      const int gd = 256 * (int)rank + 128 * g + (int)t;  // output dim
      if (p.out_bf16) {
        uint16_t* ob = reinterpret_cast<uint16_t*>(p.o) + (int64_t)bi * p.o_sb + (even ? gd : gd - 1) +
                       (int64_t)(32 * (int)ch + (even ? 0 : 1)) * p.o_sh;
        // all 16 swaps first (independent shuffles pipeline), then the 16 stores
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float a = __uint_as_float(ov[j]) * w[j], c = __uint_as_float(ov[j + 1]) * w[j + 1];
          const float r = __shfl_xor_sync(0xffffffffu, even ? c : a, 1);
          pk[j >> 1] = even ? pack_bf16x2(a, r) : pack_bf16x2(r, c);
        }
        const int h0 = 32 * (int)ch + (even ? 0 : 1);
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          if (h0 + j < p.heads) *reinterpret_cast<uint32_t*>(ob + (int64_t)j * p.o_sh) = pk[j >> 1];
      } else {
        float* ob = reinterpret_cast<float*>(p.o) + (int64_t)bi * p.o_sb + gd;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if ((int)(32 * ch) + j < p.heads) ob[(int64_t)(32 * ch + j) * p.o_sh] = __uint_as_float(ov[j]) * w[j];
      }
    }
    if (warp == 2) CTRACE(10, 2);
    GSTAMP(6);
  }
  __syncwarp();
  if (warp == 2) CTRACE(10, 4);
  GSTAMP(7);
  tc_fence_before();
  // every remote access into either CTA was awaited by its target (mbarrier phases above), so the barrier only
  // orders exits and the TMEM dealloc after both CTAs' last TMEM reads: relaxed, the O stores need not drain
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
  if (warp == 2) CTRACE(10, 5);
  if (p.trace && threadIdx.x == 64) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
    p.trace[11 * 2 * 16 + 8 * blockIdx.x + 3] = g;
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, kTmemCols);
  }
}

}  // namespace

unsigned long long* g_pair_trace = nullptr;  // loza_debug_set_pair_trace
int g_trace_cluster = 0;

bool decode_coop_eligible(const AttnProblem& a, int sms) {
  return a.sparse && a.heads >= 1 && a.heads <= kH && a.d_qk == kDqk && a.d_v == kDv && a.b % 128 == 0 &&
         2 * (int64_t)a.batch <= sms && a.n_kv < (1ll << 31);
}

bool decode_pair_dispatch(const AttnProblem& a, int32_t* status, cudaStream_t st, cudaError_t* err) {
  const int sms = device_sm_count();
  const bool coop = decode_coop_eligible(a, sms), ks = decode_ks_eligible(a, sms);
  const int k = knob(kKnobDecode);  // test override; a kernel that cannot take the problem is not forced
  if (coop && k != 2) {
    *err = launch_decode_coop(a, status, st);
    return true;
  }
  if (ks) {
    *err = launch_decode_ks(a, status, st);
    return true;
  }
  return false;
}

cudaError_t launch_decode_coop(const AttnProblem& a, int32_t* status, cudaStream_t st) {
  if (a.heads < 1 || a.heads > kH || a.d_qk != kDqk || a.d_v != kDv) return cudaErrorNotSupported;
  if (a.n_kv >= (1ll << 31)) return cudaErrorNotSupported;
  CoopParams p;
  memset(&p, 0, sizeof(p));
  p.seq_lens = a.seq_lens;
  p.batch = a.batch;
  p.heads = a.heads;
  p.s = a.s;
  p.l = a.l;
  p.b = a.b;
  p.ring = a.ring;
  p.t_cap = a.ring ? (int64_t)0x7FFFFFFF : a.n_kv;
  p.n_rows = (int32_t)a.n_kv;
  p.kraw = a.kv.seg[0].k_st == kDqk ? reinterpret_cast<const uint8_t*>(a.kv.seg[0].k) : nullptr;
  p.k_sb_bytes = a.kv.seg[0].k_sb * 2;
  p.k_st_bytes = a.kv.seg[0].k_st * 2;
  p.qraw = a.q_sh == kDqk ? reinterpret_cast<const uint8_t*>(a.q) : nullptr;
  p.q_sb_bytes = a.q_sb * 2;
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.o = a.o;
  p.o_sb = a.o_sb;
  p.o_sh = a.o_sh;
  p.out_bf16 = a.out_bf16;
  p.lse = a.lse;
  p.trace = g_pair_trace;
  p.trace_cluster = g_trace_cluster;
  p.status = status;
  const KvSeg& s = a.kv.seg[0];
  if (!encode_3d(&p.q_map, a.q, kDqk, (uint64_t)a.heads, a.batch, a.q_sh, a.q_sb, 32)) return cudaErrorInvalidValue;
  if (!encode_3d(&p.k_map, s.k, kDqk, (uint64_t)a.n_kv, a.batch, s.k_st, s.k_sb, 128)) return cudaErrorInvalidValue;
  if (!encode_4d_chunks(&p.v_map, s.v, kDv, (uint64_t)a.n_kv, a.batch, s.v_st, s.v_sb, 32, 4))
    return cudaErrorInvalidValue;
  // per launch (the attribute is per device; a process may drive several GPUs)
  cudaError_t ea = cudaFuncSetAttribute(decode_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
  if (ea != cudaSuccess) return ea;
  cudaLaunchConfig_t cfg = {};
  int nclusters = a.batch;
  if (p.kraw) {  // helper clusters on the SMs the pairs leave idle (contiguous cache rows only)
    const int spare = (device_sm_count() - 2 * a.batch) / 2;
    nclusters += spare > 0 ? (spare < kHelperClusters ? spare : kHelperClusters) : 0;
  }
  cfg.gridDim = dim3((unsigned)(2 * nclusters));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemAlloc;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, decode_coop_kernel, p);
  if (le != cudaSuccess) return le;
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza

// debug hooks (not part of include/loza.h): clock64 timeline of cluster `cluster` into dev_ptr
extern "C" void loza_debug_set_pair_trace(void* dev_ptr, int32_t cluster) {
  loza::g_pair_trace = (unsigned long long*)dev_ptr;
  loza::g_trace_cluster = cluster;
}
