// tcgen05 bf16 attention prefill over the absorbed latent MLA KV (d_qk 576, d_v 512):
// SSA (Eq. 4) and the full-attention comparator (Eq. 1).
//
// Design:
//  * CTA pair (cluster of 2, cta_group::2). One work unit = 128 consecutive query
//    rows of the [n_q*H] row space (H=64: two tokens x 64 heads); CTA r owns rows
//    64r..64r+63. Units never straddle a query block (H*b % 128 == 0), so every
//    row of a unit has the same selected key blocks: the list is the closed form
//    of the integer prologue (select_blocks.cu), computed in-kernel.
//  * An S tile is 256 keys = two 128-key sub-blocks A, B of the selected list
//    (CTA0 stages A, CTA1 stages B as the halves of the UMMA B operand). Measured on
//    B200 (tools/umma_bench.cu): a cta_group::2 UMMA costs >= ~74 cycles whatever its
//    shape, so M128 N128 runs at 43% of the tensor peak and M128 N256 at 87%; the
//    TMEM budget (O = 64 x 512 fp32 per SM) rules out M = 256, hence N = 256.
//    S = Q K^T: 36 UMMAs M128 N256 K16 (A = resident Q, 72 KB/SM); online softmax in
//    registers (a row's 256 logits live in TMEM lanes r and r+64: one max exchange);
//    P (bf16) to SMEM; O += P V: 32 UMMAs M128 N256 K16 (B = V, MN-major) into the
//    64x512 fp32 accumulator (256 TMEM columns). TMEM: O 256 + S 2 x 128 = 512 cols.
//  * Loads: TMA (SWIZZLE_128B). Two rings fed by two producer warps so K and V never
//    wait on each other: K ring 3 x 16 KB (one 128-key x 64-dim chunk per slot),
//    V ring 4 x 16 KB (64 keys x 128 dims; one commit per 4 UMMAs: a commit costs ~40 issue cycles). Both CTAs' loads complete on the leader's
//    barriers; one elected thread of the leader issues every UMMA; commits are
//    multicast to both CTAs. Q is loaded per chunk so the next unit's first S can
//    start as soon as the previous unit's last S has consumed that chunk.
//  * FA-style order S(0), S(1), PV(0), S(2), PV(1), ...: the softmax of tile t
//    overlaps PV(t-1) and S(t+1). Lazy rescaling: O and l are rescaled only when a
//    row max grows by more than 2^8 (exact; the final normalisation uses the same max).
//  * Persistent: grid = min(#units, SMs/2) clusters, units in reverse order.
#include <math.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {
using namespace sm100;

constexpr int kDqk = 576, kDv = 512, kChunks = 9;
constexpr int kThreads = 352;  // warp 0 Q/K TMA, warp 1 MMA, warps 2-9 softmax/epilogue, warp 10 V TMA
constexpr int kVWarp = 10;
constexpr int kKSlots = 3;
constexpr int kKSlotBytes = 16384;  // 128 keys x 64 dims
constexpr int kVKeys = 64;                 // keys per V slab
constexpr int kVSlots = 4;
constexpr int kVSlotBytes = kVKeys * 256;  // kVKeys keys x 128 dims (two 64-dim column blocks)
constexpr int kVGroups = 256 / kVKeys;     // slabs per 256-key tile and N-half
constexpr int kQBytes = kChunks * 64 * 128;  // 73728 per CTA
constexpr int kPBytes = 4 * 64 * 128;        // 32768: 4 key chunks (64 keys) x 64 rows
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffK = kOffP + kPBytes;
constexpr int kOffV = kOffK + kKSlots * kKSlotBytes;
constexpr int kOffBar = kOffV + kVSlots * kVSlotBytes;  // 229376
constexpr int kBarKFull = 0;
constexpr int kBarKEmpty = kBarKFull + kKSlots;
constexpr int kBarVFull = kBarKEmpty + kKSlots;
constexpr int kBarVEmpty = kBarVFull + kVSlots;
constexpr int kBarQFull = kBarVEmpty + kVSlots;  // [9] per Q chunk
constexpr int kBarQEmpty = kBarQFull + kChunks;  // [9]
constexpr int kBarSFull = kBarQEmpty + kChunks;  // [2]
constexpr int kBarSFree = kBarSFull + 2;         // [2]
constexpr int kBarPFull = kBarSFree + 2;         // [1]
constexpr int kBarOFull = kBarPFull + 1;         // [2]
constexpr int kBarOFree = kBarOFull + 2;
constexpr int kNumBars = kBarOFree + 1;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffRed = (kOffTmemPtr + 4 + 15) & ~15;  // float [2 buf][4 quarter-rows][64]; epilogue reuses it
constexpr int kSmemUsed = kOffRed + 2 * 4 * 64 * 4;
// The dynamic smem base is 1024-byte aligned (no static smem; checked at run time), so no slack.
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 0, kTmemS = 256;  // S buffer b at 256 + 128 b
constexpr uint32_t kSoftmaxWarps = 8;
constexpr uint32_t kArrivalsPerPair = 2 * kSoftmaxWarps;

struct PrefillParams {
  CUtensorMap q_map;
  CUtensorMap k_map[3];
  CUtensorMap v_map[3];
  int64_t seg_begin[3];
  int32_t seg_len[3];
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
  unsigned long long* trace;  // debug timeline (cluster 0, leader CTA), NULL in production
};

struct Unit {
  int32_t bi;
  int64_t row0;            // first row of the unit in the batch's [n_q*H] rows
  int64_t tok_lo, tok_hi;  // absolute positions
  int32_t n_sink, loc_begin, n128, n_tiles;  // 128-key sub-blocks; 256-key S tiles
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
// start key of the j-th selected 128-key sub-block, or -1 if j is past the list
__device__ __forceinline__ int64_t sub_k0(const Unit& U, int j) {
  if (j >= U.n128) return -1;
  return (int64_t)(j < U.n_sink ? j : U.loc_begin + (j - U.n_sink)) * 128;
}
__device__ __forceinline__ int seg_of(const PrefillParams& p, int64_t k0) {
  int s = 0;
  if (p.nseg > 1 && k0 >= p.seg_begin[1]) s = 1;
  if (p.nseg > 2 && k0 >= p.seg_begin[2]) s = 2;
  return s;
}
// (segment, row coordinate) of the sub-block at k0 (+ off rows); a missing sub-block maps to an
// out-of-bounds box (TMA fills zeros, so its masked keys contribute 0 * 0)
__device__ __forceinline__ void kv_coord(const PrefillParams& p, int64_t k0, int32_t off, int& sg, int32_t& row) {
  if (k0 < 0) {
    sg = 0;
    row = p.seg_len[0];
    return;
  }
  sg = seg_of(p, k0);
  row = (int32_t)(k0 - p.seg_begin[sg]) + off;
}
__device__ __forceinline__ int64_t unit_index(const PrefillParams& p, int64_t it) {
  return p.total_units - 1 - it;  // heaviest (latest rows) first
}

#define TRACE(slot, idx)                                                                        \
  do {                                                                                          \
    if (p.trace && cid == 0 && rank == 0 && (idx) < 64 && lane == 0) p.trace[(slot)*64 + (idx)] = clock64(); \
  } while (0)

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    prefill_tc_kernel(const __grid_constant__ PrefillParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();  // SWIZZLE_128B tiles need a 1024-byte aligned base
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* red = reinterpret_cast<float*>(smem + kOffRed);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kKSlots; ++i) {
      mbar_init(bar(kBarKFull + i), 1);
      mbar_init(bar(kBarKEmpty + i), 1);
    }
    for (int i = 0; i < kVSlots; ++i) {
      mbar_init(bar(kBarVFull + i), 1);
      mbar_init(bar(kBarVEmpty + i), 1);
    }
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

  // Producer and MMA roles run with the whole warp (warp-uniform control flow keeps the
  // descriptors / coordinates in uniform registers); one elected lane issues each TMA / UMMA.
  // A lane-0-guarded issue loop made ptxas emit an R2UR "uniformisation loop" per UMMA,
  // which capped the issue rate at ~40% of the tensor pipe (tools/umma_interf.cu).
  if (warp == 0) {
    // ===================================================== Q + K TMA producer (both CTAs)
    const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_last();
    uint32_t uc = 0, kc = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = make_unit(p, unit_index(p, it));
      for (int c = 0; c < kChunks; ++c) {
        mbar_wait(bar(kBarQEmpty + c), (uc & 1) ^ 1);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarQFull + c), 2 * 8192);
          tma_load_3d_pair(sbase + kOffQ + c * 8192, &p.q_map, c * 64, (int32_t)(U.row0 + 64 * rank), U.bi,
                           mapa(bar(kBarQFull + c), 0), pol_q);
        }
        __syncwarp();
      }
      for (int i = 0; i < U.n_tiles; ++i) {
        int sg;
        int32_t row;
        kv_coord(p, sub_k0(U, 2 * i + (int)rank), 0, sg, row);  // CTA r stages sub-block 2i+r
        for (int c = 0; c < kChunks; ++c, ++kc) {
          const uint32_t slot = kc % kKSlots;
          mbar_wait(bar(kBarKEmpty + slot), ((kc / kKSlots) & 1) ^ 1);
          if (elect_one()) {
            if (rank == 0) mbar_arrive_expect_tx(bar(kBarKFull + slot), 2 * kKSlotBytes);
            tma_load_3d_pair(sbase + kOffK + slot * kKSlotBytes, &p.k_map[sg], c * 64, row, U.bi,
                             mapa(bar(kBarKFull + slot), 0), pol_kv);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == kVWarp) {
    // ===================================================== V TMA producer (both CTAs)
    const uint64_t pol_kv = policy_evict_last();
    uint32_t vc = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl) {
      const Unit U = make_unit(p, unit_index(p, it));
      for (int i = 0; i < U.n_tiles; ++i) {
        for (int kg = 0; kg < kVGroups; ++kg) {  // kVKeys-key groups: first half sub-block A, second half B
          int sg;
          int32_t row;
          kv_coord(p, sub_k0(U, 2 * i + kg / (kVGroups / 2)), kVKeys * (kg % (kVGroups / 2)), sg, row);
          for (int nh = 0; nh < 2; ++nh, ++vc) {
            const uint32_t slot = vc % kVSlots;
            mbar_wait(bar(kBarVEmpty + slot), ((vc / kVSlots) & 1) ^ 1);
            if (elect_one()) {
              if (rank == 0) mbar_arrive_expect_tx(bar(kBarVFull + slot), 2 * kVSlotBytes);
              const uint32_t fb = mapa(bar(kBarVFull + slot), 0);
              for (int e = 0; e < 2; ++e)
                tma_load_3d_pair(sbase + kOffV + slot * kVSlotBytes + e * (kVKeys * 128), &p.v_map[sg],
                                 256 * nh + 128 * (int)rank + 64 * e, row, U.bi, fb, pol_kv);
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer (leader CTA only)
    if (rank == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 256, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 256, false, true);
      const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);  // Q chunk c, K step k: + (8192c + 32k) >> 4
      const uint64_t dk = sdesc_sw128(sbase + kOffK, 16, 1024);  // K slot j: + 16384 j >> 4
      const uint64_t dp = sdesc_sw128(sbase + kOffP, 16, 1024);  // P chunk: + 8192 chunk >> 4
      const uint64_t dv = sdesc_sw128(sbase + kOffV, kVKeys * 128, 1024);  // V slot j (MN-major)
      uint32_t uc = 0, g = 0, kc = 0, vc = 0;
      long long kwait = 0, vwait = 0;
      auto issue_s = [&](uint32_t gi, bool first, bool last) {
        const uint32_t buf = gi & 1;
        kwait = 0;
        TRACE(0, gi);
        mbar_wait(bar(kBarSFree + buf), ((gi >> 1) & 1) ^ 1);
        TRACE(1, gi);
        tc_fence_after();
        const uint32_t d = tmem + kTmemS + 128 * buf;
        for (int c = 0; c < kChunks; ++c, ++kc) {
          const uint32_t slot = kc % kKSlots;
          const long long w0 = clock64();
          if (first) mbar_wait(bar(kBarQFull + c), uc & 1);
          mbar_wait(bar(kBarKFull + slot), (kc / kKSlots) & 1);
          kwait += clock64() - w0;
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16_pair(d, dq + (uint64_t)((8192 * c + 32 * k) >> 4),
                             dk + (uint64_t)((kKSlotBytes * slot + 32 * k) >> 4), idesc_s, (c | k) != 0);
            umma_commit_pair_mc(bar(kBarKEmpty + slot), 3);
            if (last) umma_commit_pair_mc(bar(kBarQEmpty + c), 3);
          }
          __syncwarp();
        }
        if (elect_one()) umma_commit_pair_mc(bar(kBarSFull + buf), 3);
        __syncwarp();
        TRACE(2, gi);
        if (p.trace && cid == 0 && gi < 64 && lane == 0) p.trace[11 * 64 + gi] = kwait;
      };
      auto issue_pv = [&](uint32_t gi, bool first) {
        TRACE(3, gi);
        vwait = 0;
        mbar_wait(bar(kBarPFull), gi & 1);
        if (first && uc > 0) mbar_wait(bar(kBarOFree), (uc - 1) & 1);
        TRACE(4, gi);
        tc_fence_after();
        for (int kg = 0; kg < kVGroups; ++kg)
          for (int nh = 0; nh < 2; ++nh, ++vc) {
            const uint32_t slot = vc % kVSlots;
            const long long w0 = clock64();
            mbar_wait(bar(kBarVFull + slot), (vc / kVSlots) & 1);
            vwait += clock64() - w0;
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < kVKeys / 16; ++kk) {
                const int key = kg * kVKeys + 16 * kk;  // key of the 256-key tile (P column)
                umma_bf16_pair(tmem + kTmemO + 128 * nh, dp + (uint64_t)((8192 * (key >> 6) + 2 * (key & 63)) >> 4),
                               dv + (uint64_t)((kVSlotBytes * slot + 2048 * kk) >> 4), idesc_pv,
                               !(first && kg == 0 && kk == 0));
              }
              umma_commit_pair_mc(bar(kBarVEmpty + slot), 3);
            }
            __syncwarp();
          }
        if (elect_one()) umma_commit_pair_mc(bar(kBarOFull + (gi & 1)), 3);
        __syncwarp();
        TRACE(5, gi);
        if (p.trace && cid == 0 && gi < 64 && lane == 0) p.trace[12 * 64 + gi] = vwait;
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
    // TMEM lane quarter = warp % 4; lane tl holds row r = tl % 64 and the 128 logits of sub-block kh = tl / 64.
    // Warps 2-5 take columns [0, 64) of those 128 (ch = 0), warps 6-9 columns [64, 128) (ch = 1), so each
    // row's 256 logits are spread over 4 threads (quarter q = 2 kh + ch) and 2 warps share each sub-partition.
    const uint32_t wq = warp & 3;
    const uint32_t ch = (warp - 2) >> 2;
    const uint32_t tl = wq * 32 + lane;
    const uint32_t r = tl & 63, kh = tl >> 6, q4 = 2 * kh + ch;
    const uint32_t taddr = tmem + ((wq * 32) << 16);
    const uint32_t sfree0 = mapa(bar(kBarSFree), 0), pfull = mapa(bar(kBarPFull), 0), ofree = mapa(bar(kBarOFree), 0);
    const float ln2 = 0.69314718055994531f;
    const int64_t rows_b = (int64_t)p.n_q * p.heads;
    const float sl2 = p.scale_log2;
    const int causal = p.causal;
    const int64_t n_kv = p.n_kv;
    constexpr uint32_t kSmThreads = 32 * kSoftmaxWarps;
    uint32_t g = 0, uc = 0;
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = make_unit(p, unit_index(p, it));
      const int64_t row_g = U.row0 + 64 * rank + r;
      const bool row_ok = row_g < rows_b;
      const int64_t my_tok = p.q_start + (row_ok ? row_g : rows_b - 1) / p.heads;
      float m_used = -INFINITY, lrow = 0.f;
      for (int i = 0; i < U.n_tiles; ++i) {
        const uint32_t gi = g + i, buf = gi & 1;
        const int64_t kb0 = sub_k0(U, 2 * i + (int)kh);  // this thread's sub-block (-1: none)
        // number of valid keys among this thread's 64 columns [kb0 + 64 ch, +64): causal, tail, missing block
        int32_t nvalid = 64;
        if (kb0 < 0) {
          nvalid = 0;
        } else {
          const int64_t c0 = kb0 + 64 * ch;
          int64_t lim = n_kv - c0;
          if (causal && my_tok + 1 - c0 < lim) lim = my_tok + 1 - c0;
          nvalid = lim < 0 ? 0 : (lim > 64 ? 64 : (int32_t)lim);
        }
        if (warp == 2 && lane == 0) TRACE(6, gi);
        mbar_wait(bar(kBarSFull + buf), (gi >> 1) & 1);
        if (warp == 2 && lane == 0) TRACE(7, gi);
        tc_fence_after();
        const uint32_t sa = taddr + kTmemS + 128 * buf + 64 * ch;
        uint32_t v[64];
        tmem_ld32(sa, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld32(sa + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(sfree0 + 8 * buf);  // S columns of this warp are in registers
        if (nvalid < 64) {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (j >= nvalid) v[j] = __float_as_uint(-INFINITY);
        }
        // row max (raw logits; scale > 0 commutes with max), 4 independent chains
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
        // P = exp2(s * scale - m): 4 independent partial sums; packed to bf16 pairs
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
        // PV(t-1) must be complete before O is rescaled and before P (single buffer) is overwritten
        if (i > 0) {
          const uint32_t gp = gi - 1;
          if (warp == 2 && lane == 0) TRACE(8, gi);
          mbar_wait(bar(kBarOFull + (gp & 1)), (gp >> 1) & 1);
          if (warp == 2 && lane == 0) TRACE(9, gi);
          tc_fence_after();
          if (__any_sync(0xffffffffu, resc)) {
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {  // this warp's O columns [128 ch, 128 ch + 128)
              uint32_t ov[32];
              tmem_ld32(taddr + kTmemO + 128 * ch + 32 * c, ov);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr);
              tmem_st32(taddr + kTmemO + 128 * ch + 32 * c, ov);
            }
            tmem_wait_st();
          }
        }
        // P chunk q4 (keys 64 q4 .. of the 256-key tile), row r: one 128-byte swizzled row
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
        if (warp == 2 && lane == 0) TRACE(10, gi);
      }
      // ---------------- epilogue: O / l -> global (this warp: O columns [128 ch, +128) = dims 256 ch + 128 kh ..)
      const uint32_t gl = g + U.n_tiles - 1;
      mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
      tc_fence_after();
      float* ls = red + ((gl + 1) & 1) * 256;  // the exchange buffer not used by the last tile
      ls[q4 * 64 + r] = lrow;
      named_bar_sync(1, kSmThreads);
      const float ltot = (ls[r] + ls[64 + r]) + (ls[128 + r] + ls[192 + r]);
      const float inv = 1.0f / ltot;
      named_bar_sync(1, kSmThreads);  // everyone has read ls before the next unit's first exchange writes red
      char* obase = reinterpret_cast<char*>(p.o) +
                    ((int64_t)U.bi * p.o_sb + (row_ok ? row_g : 0) * kDv) * (p.out_bf16 ? 2 : 4);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        tmem_ld32(taddr + kTmemO + 128 * ch + 32 * c, ov);
        tmem_wait_ld();
        const int dim0 = 256 * (int)ch + 128 * (int)kh + 32 * c;
        if (row_ok) {
          if (p.out_bf16) {
            uint32_t w[16];
#pragma unroll
            for (int j = 0; j < 16; ++j)
              w[j] = pack_bf16x2(__uint_as_float(ov[2 * j]) * inv, __uint_as_float(ov[2 * j + 1]) * inv);
            char* dst = obase + dim0 * 2;
#pragma unroll
            for (int q = 0; q < 4; ++q) st_global_v4(dst + 16 * q, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
          } else {
            char* dst = obase + dim0 * 4;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              st_global_v4(dst + 16 * q, __float_as_uint(__uint_as_float(ov[4 * q]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 1]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 2]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 3]) * inv));
          }
        }
      }
      if (p.lse && row_ok && q4 == 0) {
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

unsigned long long* g_debug_trace = nullptr;

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
  p.trace = g_debug_trace;
  p.total_units = p.units_per_batch * a.batch;
  if (p.total_units == 0) return cudaSuccess;
  if (!encode_3d(&p.q_map, a.q, kDqk, rows, a.batch, kDqk, a.q_sb, 64)) return cudaErrorInvalidValue;
  p.nseg = a.kv.nseg;
  for (int i = 0; i < a.kv.nseg; ++i) {
    const KvSeg& s = a.kv.seg[i];
    p.seg_begin[i] = s.pos_begin;
    const uint64_t len = (uint64_t)(s.pos_end - s.pos_begin);
    p.seg_len[i] = (int32_t)len;
    if (!encode_3d(&p.k_map[i], s.k, kDqk, len, a.batch, s.k_st, s.k_sb, 128)) return cudaErrorInvalidValue;
    if (!encode_3d(&p.v_map[i], s.v, kDv, len, a.batch, s.v_st, s.v_sb, kVKeys)) return cudaErrorInvalidValue;
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

// debug hook (not part of include/loza.h): record a clock64 timeline of cluster 0 into dev_ptr[11*64]
extern "C" void loza_debug_set_trace(void* dev_ptr) { loza::g_debug_trace = (unsigned long long*)dev_ptr; }
