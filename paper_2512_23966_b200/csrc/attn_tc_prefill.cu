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
//  * Loads: TMA (SWIZZLE_128B) into ONE ring of 3 x 32 KB slots consumed in UMMA order
//    (K(0), K(1), V(0), K(2), V(1), ..., V(T-1) per unit): a K item is 128 keys x 2 dim chunks
//    (4-D box), a V item one 128-key sub-block x 128 dims (4-D box); the RoPE chunk 8 of K has
//    a one-slot ring of its own. 32 KB items halve the per-item cost on the MMA warp (a wait on a
//    full barrier ~64 issue cycles, a commit ~40 tensor-pipe cycles; tools/umma_interf.cu) versus
//    16 KB items. Warp 0 issues the Q and K items, warp 10 the V items of the same sequence, with
//    a position handshake so mbarrier parities cannot alias (see acquire()). A lean issue loop
//    reaches ~100 B/clk/SM from L2 (tools/tma_box.cu); the fill rate is bound by bytes in flight,
//    i.e. by the ring size (SMEM: Q 72 KB + P 32 KB + ring 96 + 16 KB). Both CTAs' loads complete
//    on the leader's barriers; one elected thread of the leader issues every UMMA; commits are
//    multicast to both CTAs. Q is loaded per chunk so the next unit's first S can start as soon
//    as the previous unit's last S has consumed that chunk.
//  * Epilogue: O -> registers (then O is released to the next unit's PV), bf16, staged in the
//    P buffer as [64 x 64] swizzled boxes, TMA tensor stores (st.global from 256 threads stalled
//    the MMA warp's barrier traffic at every unit boundary: +12% end to end when removed).
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

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
#ifndef DOHAT_L1
#define DOHAT_L1 1  // d_o_hat loads allocate in L1 (a thread's 4 x 16 B of one 64-B run share 2 sectors)
#endif
__device__ __forceinline__ uint4 ldg_nc_v4(const void* ptr) {
  uint4 r;
#if DOHAT_L1
  asm volatile("ld.global.nc.L1::evict_first.v4.u32 {%0,%1,%2,%3}, [%4];"
#else
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
#endif
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr));
  return r;
}
#define FULL_L(slot) (full_l + 8 * (slot))
#define QFULL_L(c) (qfull_l + 8 * (c))
constexpr int kDqk = 576, kDv = 512, kChunks = 9;
constexpr int kThreads = 352;  // warp 0 Q/K TMA, warp 1 MMA, warps 2-9 softmax/epilogue, warp 10 V TMA
constexpr int kVWarp = 10;
constexpr int kSlots = 3;
constexpr int kSlotBytes = 32768;
constexpr int kChunkBytes = 16384;         // 128 keys x 64 dims
constexpr int kKItems = 4;                 // big-ring K items per tile: chunks {0,1} {2,3} {4,5} {6,7};
                                           // chunk 8 (RoPE) goes through its own one-slot ring
constexpr int kVKeys = 128;                // V item: one 128-key sub-block x 128 dims (two 64-dim chunks)
constexpr int kVGroups = 256 / kVKeys;     // V items per tile and N-half
constexpr int kVItems = 2 * kVGroups;      // V items per tile
static_assert(kVKeys * 256 == kSlotBytes, "one slot size");
constexpr int kQBytes = kChunks * 64 * 128;  // 73728 per CTA
constexpr int kPBytes = 4 * 64 * 128;        // 32768: 4 key chunks (64 keys) x 64 rows
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kQBytes;
constexpr int kOffRing = kOffP + kPBytes;
constexpr int kOffRope = kOffRing + kSlots * kSlotBytes;  // 204800: K chunk 8 of the next S
constexpr int kOffBar = kOffRope + kChunkBytes;            // 221184
constexpr int kBarFull = 0;
constexpr int kBarEmpty = kBarFull + kSlots;
constexpr int kBarRopeFull = kBarEmpty + kSlots;
constexpr int kBarRopeEmpty = kBarRopeFull + 1;
constexpr int kBarQFull = kBarRopeEmpty + 1;  // [9] per Q chunk
constexpr int kBarQEmpty = kBarQFull + kChunks;  // [9]
constexpr int kBarSFull = kBarQEmpty + kChunks;  // [2]
constexpr int kBarSFree = kBarSFull + 2;         // [2]
constexpr int kBarPFull = kBarSFree + 2;         // [1]
constexpr int kBarOFull = kBarPFull + 1;         // [2]
constexpr int kBarOFree = kBarOFull + 2;
constexpr int kBarOfFull = kBarOFree + 1;   // calibration: O_full of the unit staged in the Q region (local)
// calibration: the epilogue has read the O_full box in Q chunk slot c ([8]; the 2 warps that read it, local)
constexpr int kBarOfEmpty = kBarOfFull + 1;
constexpr int kNumBars = kBarOfEmpty + 8;
// O_full box m (dims 64 m ..) lives in Q chunk slot of_slot(m): the boxes the epilogue finishes first (its
// warps' first 64 dims, m even) take slots 0-3, so the next unit's Q chunks 0-3 -- and the S UMMAs on them --
// can start while the epilogue still works on the other half
__host__ __device__ constexpr int of_slot(int m) { return (m & 1) * 4 + (m >> 1); }
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffPub = kOffTmemPtr + 4;                // uint32 [2]: producers' next ring positions
constexpr int kOffRed = (kOffPub + 8 + 15) & ~15;  // float [2 buf][4 quarter-rows][64]; epilogue reuses it
constexpr int kSmemUsed = kOffRed + 2 * 4 * 64 * 4;
// The dynamic smem base is 1024-byte aligned (no static smem; checked at run time), so no slack.
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 0, kTmemS = 256;  // S buffer b at 256 + 128 b
constexpr uint32_t kSoftmaxWarps = 8;
constexpr uint32_t kArrivalsPerPair = 2 * kSoftmaxWarps;

#ifndef MLA_SOFTMAX_V2
#define MLA_SOFTMAX_V2 1
#endif

struct PrefillParams {
  CUtensorMap q_map;
  CUtensorMap k_map[3];   // 3-D, box 128 rows x 1 chunk (the RoPE chunk 8)
  CUtensorMap k2_map[3];  // 4-D, box 128 rows x 2 chunks
  CUtensorMap v_map[3];   // 4-D, box 128 rows x 2 chunks
  CUtensorMap o_map;      // bf16 output, box 64 rows x 64 dims (TMA-store epilogue)
  CUtensorMap of_map;     // calibration: O_full, same boxes (staged in the Q region for the epilogue)
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
  int64_t lse_sh;  // lse head stride (elements)
  int64_t units_per_batch, total_units;
  // fused calibration forward (Eq. 3 in the epilogue; CalibArgs): o receives o_hat
  const uint8_t* o_full;   // NULL: plain prefill
  const uint8_t* d_o_hat;  // NULL: forward only
  const float* alpha;
  double* part;            // per-CTA fp64 partial of d_alpha
  int32_t* status;
  int32_t small;              // all index math fits in 31 bits (make_unit fast path)
  FastDiv div_upb, div_heads, div_b;  // multiply-shift divisors for the small path
  unsigned long long* trace;  // debug timeline (cluster 0, leader CTA), NULL in production
};

struct Unit {
  int32_t bi;
  int64_t row0;            // first row of the unit in the batch's [n_q*H] rows
  int64_t tok_lo, tok_hi;  // absolute positions
  int32_t n_sink, loc_begin, n128, n_tiles;  // 128-key sub-blocks; 256-key S tiles
};

// Index math in T: uint32_t when every quantity fits (PrefillParams::small, the common case) -- the
// 64-bit divisions of the general path cost ~1.4K cycles per unit on the MMA warp's critical path.
template <typename T>
__device__ __forceinline__ Unit make_unit_t(const PrefillParams& p, int64_t u64) {
  Unit U;
  constexpr bool fast = sizeof(T) == 4;
  const T u = (T)u64, upb = (T)p.units_per_batch, heads = (T)p.heads;
  const T bi = fast ? (T)p.div_upb.div((uint32_t)u) : u / upb;
  const T row0 = (u - bi * upb) * 128;
  const T rows = (T)p.n_q * heads;
  T rlast = row0 + 127;
  if (rlast > rows - 1) rlast = rows - 1;
  U.bi = (int32_t)bi;
  U.row0 = (int64_t)row0;
  const T tok_lo = (T)p.q_start + (fast ? (T)p.div_heads.div((uint32_t)row0) : row0 / heads),
          tok_hi = (T)p.q_start + (fast ? (T)p.div_heads.div((uint32_t)rlast) : rlast / heads);
  U.tok_lo = (int64_t)tok_lo;
  U.tok_hi = (int64_t)tok_hi;
  const T last_sub = p.causal ? tok_hi / 128 : ((T)p.n_kv - 1) / 128;
  if (!p.sparse) {
    U.n_sink = 0;
    U.loc_begin = 0;
    U.n128 = (int32_t)(last_sub + 1);
  } else {
    const int64_t tpb = p.b / 128, QB = (int64_t)(fast ? (T)p.div_b.div((uint32_t)tok_lo) : tok_lo / (T)p.b);
    int64_t sink_end = (QB + 1 < p.s ? QB + 1 : p.s) * tpb;
    if (sink_end > (int64_t)last_sub + 1) sink_end = (int64_t)last_sub + 1;
    int64_t lb = QB - p.l + 1;
    if (lb < p.s) lb = p.s;
    lb *= tpb;
    int64_t le = (QB + 1) * tpb;
    if (le > (int64_t)last_sub + 1) le = (int64_t)last_sub + 1;
    U.n_sink = (int32_t)sink_end;
    U.loc_begin = (int32_t)lb;
    U.n128 = (int32_t)(sink_end + (le > lb ? le - lb : 0));
  }
  U.n_tiles = (U.n128 + 1) / 2;
  return U;
}
__device__ __forceinline__ Unit make_unit(const PrefillParams& p, int64_t u) {
  return p.small ? make_unit_t<uint32_t>(p, u) : make_unit_t<int64_t>(p, u);
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

// kMode 1, 2: fused calibration forward (Eq. 3 in the epilogue), 2 with d_alpha from d_o_hat; separate
// instantiations so the plain prefill and the forward-only blend keep their own register allocation
template <int kMode>
__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    prefill_tc_kernel(const __grid_constant__ PrefillParams p) {
  constexpr bool kCalib = kMode >= 1, kDoHat = kMode == 2;
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
    mbar_init(bar(kBarOfFull), 1);
    for (int i = 0; i < 8; ++i) mbar_init(bar(kBarOfEmpty + i), 2);
    reinterpret_cast<volatile uint32_t*>(smem + kOffPub)[0] = 0;
    reinterpret_cast<volatile uint32_t*>(smem + kOffPub)[1] = 0;
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&p.q_map);
    for (int i = 0; i < p.nseg; ++i) {
      prefetch_tmap(&p.k_map[i]);
      prefetch_tmap(&p.k2_map[i]);
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
  // Ring position -> (slot, phase), advanced incrementally (no divisions on the issue path).
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
  // Two producers share the ring. A parity wait on empty[slot] for use j is only sound once use j-1 of
  // that slot has passed its own wait (else the barrier may be two phases behind and the parity aliases).
  // When use j-1 belongs to the other producer this is not implied by program order, so each producer
  // publishes the ring position of its next item (all its items before it are issued) and waits until
  // the other's published position passes pos - kSlots. No deadlock: everything before the other's
  // published position is issued, so it can always advance.
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
    uint32_t uc = 0;
    uint32_t gk = 0;
    auto no_hook = [](int) {};
    auto load_k = [&](const Unit& U, int i, auto&& before_item) {
      int sg;
      int32_t row;
      kv_coord(p, sub_k0(U, 2 * i + (int)rank), 0, sg, row);  // CTA r stages sub-block 2i+r
      // chunk 8 first: its slot was freed by the previous S, long before this one needs it
      mbar_wait(bar(kBarRopeEmpty), (gk & 1) ^ 1);
      if (elect_one()) {
        if (rank == 0) mbar_arrive_expect_tx(bar(kBarRopeFull), 2 * kChunkBytes);
        tma_load_3d_pair(sbase + kOffRope, &p.k_map[sg], 8 * 64, row, U.bi, rope_l, pol_kv);
      }
      __syncwarp();
      for (int j = 0; j < kKItems; ++j, rp.step()) {
        before_item(j);
        acquire(rp, 0);
        if (j == 0) TRACE(13, gk);
        if (j == kKItems - 1) TRACE(14, gk);
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + rp.slot), 2 * kSlotBytes);
          tma_load_4d_pair(ring + rp.slot * kSlotBytes, &p.k2_map[sg], 0, row, 2 * j, U.bi, FULL_L(rp.slot), pol_kv);
        }
        __syncwarp();
      }
      ++gk;
    };
    // calibration: once a unit's last S has released the Q region, the unit's O_full rows are staged there
    // (8 boxes [64 rows x 64 dims], TMA) for the epilogue; the next unit's Q follows the epilogue's release
    Unit Uprev;
    auto stage_o_full = [&](const Unit& Us, uint32_t ucs) {
      for (int c = 0; c < kChunks; ++c) mbar_wait(bar(kBarQEmpty + c), ucs & 1);  // unit ucs's last S is done
      if (elect_one()) {
        mbar_arrive_expect_tx(bar(kBarOfFull), 8 * 8192);
        for (int m = 0; m < 8; ++m)
          tma_load_3d(sbase + kOffQ + of_slot(m) * 8192, &p.of_map, 64 * m, (int32_t)(Us.row0 + 64 * rank), Us.bi,
                      bar(kBarOfFull), pol_q);
      }
      __syncwarp();
    };
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = make_unit(p, unit_index(p, it));
      // Before blocking outside acquire(): publish the next ring position (all items before it are issued or
      // the V producer's), else the V producer's handshake for the previous unit's last V items waits on this
      // warp while this warp waits (here, or in the calibration OfEmpty wait) on work that needs those items.
      if (lane == 0) pub[0] = rp.pos;
      __syncwarp();
      if constexpr (kCalib) {
        if (uc > 0) stage_o_full(Uprev, uc - 1);
        // d_o_hat rows of this unit into L2 ahead of the epilogue (read with plain loads there; an L2
        // prefetch of the O_full rows as well measured slower)
        {
          const int64_t r0 = U.row0 + 64 * rank, rows_b = (int64_t)p.n_q * p.heads;
          const int64_t nl = ((rows_b - r0 < 64 ? rows_b - r0 : 64) * kDv * 2) / 128;
          const int64_t off = ((int64_t)U.bi * p.o_sb + r0 * kDv) * 2;
          for (int64_t ln = lane; ln < nl; ln += 32) {
            if (p.d_o_hat) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p.d_o_hat + off + ln * 128));
          }
        }
      }
      auto load_q = [&](int c) {
        mbar_wait(bar(kBarQEmpty + c), (uc & 1) ^ 1);
        if (kCalib && uc > 0 && c < 8) {  // the previous unit's epilogue has read the O_full box in this slot
          if (lane == 0) pub[0] = rp.pos;
          __syncwarp();
          mbar_wait(bar(kBarOfEmpty + c), (uc - 1) & 1);
        }
        if (elect_one()) {
          if (rank == 0) mbar_arrive_expect_tx(bar(kBarQFull + c), 2 * 8192);
          tma_load_3d_pair(sbase + kOffQ + c * 8192, &p.q_map, c * 64, (int32_t)(U.row0 + 64 * rank), U.bi,
                           QFULL_L(c), pol_q);
        }
        __syncwarp();
      };
      if constexpr (kCalib) {
        // Q chunk 8 (no O_full there), then each chunk pair as its slots are released, interleaved with the
        // first tile's K items so the S UMMAs on chunks 0-3 overlap the previous unit's epilogue
        load_q(8);
        load_k(U, 0, [&](int j) {
          load_q(2 * j);
          load_q(2 * j + 1);
        });
        Uprev = U;
      } else {
        for (int c = 0; c < kChunks; ++c) load_q(c);
        load_k(U, 0, no_hook);
      }
      for (int i = 1; i < U.n_tiles; ++i) {
        load_k(U, i, no_hook);
        rp.skip(kVItems);  // V(i-1): warp kVWarp
      }
      rp.skip(kVItems);
    }
    if (lane == 0) pub[0] = 0xFFFFFFFFu;
    if constexpr (kCalib) {
      if (uc > 0) stage_o_full(Uprev, uc - 1);
    }
  } else if (warp == kVWarp) {
    // ===================================================== V items producer (both CTAs)
    const uint64_t pol_kv = policy_evict_last();
    const uint32_t full_l = mapa(bar(kBarFull), 0);
    const uint32_t ring = sbase + kOffRing;
    RingPos rp;
    uint32_t gv = 0;
    auto load_v = [&](const Unit& U, int i) {
      for (int kg = 0; kg < kVGroups; ++kg) {  // sub-block A then B of tile i
        int sg;
        int32_t row;
        kv_coord(p, sub_k0(U, 2 * i + kg), 0, sg, row);
        for (int nh = 0; nh < 2; ++nh, rp.step()) {
          acquire(rp, 1);
          if (kg == 0 && nh == 0) TRACE(15, gv);
          if (kg == 1 && nh == 1) TRACE(16, gv);
          if (elect_one()) {
            if (rank == 0) mbar_arrive_expect_tx(bar(kBarFull + rp.slot), 2 * kSlotBytes);
            // dims [256 nh + 128 r, +128) = column chunks 4 nh + 2 r, +1 (one 4-D box)
            tma_load_4d_pair(ring + rp.slot * kSlotBytes, &p.v_map[sg], 0, row, 4 * nh + 2 * (int)rank, U.bi,
                             FULL_L(rp.slot), pol_kv);
          }
          __syncwarp();
        }
      }
      ++gv;
    };
    for (int64_t it = cid; it < n_iter_total; it += ncl) {
      const Unit U = make_unit(p, unit_index(p, it));
      rp.skip(kKItems);  // K(0)
      for (int i = 1; i < U.n_tiles; ++i) {
        rp.skip(kKItems);  // K(i)
        load_v(U, i - 1);
      }
      load_v(U, U.n_tiles - 1);
    }
    if (lane == 0) pub[1] = 0xFFFFFFFFu;
  } else if (warp == 1) {
    // ===================================================== MMA issuer (leader CTA only)
    if (rank == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 256, false, false);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 256, false, true);
      const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);  // Q chunk c, K step k: + (8192c + 32k) >> 4
      const uint64_t dk = sdesc_sw128(sbase + kOffRing, 16, 1024);  // ring slot j, chunk cc: + (32768 j + 16384 cc) >> 4
      const uint64_t dp = sdesc_sw128(sbase + kOffP, 16, 1024);  // P chunk: + 8192 chunk >> 4
      const uint64_t dv = sdesc_sw128(sbase + kOffRing, kVKeys * 128, 1024);  // ring slot j as a V item (MN-major,
                                                                              // 64-dim chunks kVKeys*128 B apart)
      uint32_t uc = 0, g = 0;
      RingPos rp;
      long long kwait = 0, vwait = 0;
      auto issue_s = [&](uint32_t gi, bool first, bool last) {
        const uint32_t buf = gi & 1;
        kwait = 0;
        TRACE(0, gi);
        mbar_wait(bar(kBarSFree + buf), ((gi >> 1) & 1) ^ 1);
        TRACE(1, gi);
        tc_fence_after();
        const uint32_t d = tmem + kTmemS + 128 * buf;
        for (int j = 0; j <= kKItems; ++j) {  // big items j < 4 (chunks 2j, 2j+1), then the RoPE chunk
          const bool rope = j == kKItems;
          const uint32_t slot = rp.slot;
          const int nc = rope ? 1 : 2;
          const long long w0 = clock64();
          if (first) {
            mbar_wait(bar(kBarQFull + 2 * j), uc & 1);
            if (nc == 2) mbar_wait(bar(kBarQFull + 2 * j + 1), uc & 1);
          }
          if (rope)
            mbar_wait(bar(kBarRopeFull), gi & 1);
          else
            mbar_wait(bar(kBarFull + slot), rp.phase);
          kwait += clock64() - w0;
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
          for (int nh = 0; nh < 2; ++nh, rp.step()) {
            const uint32_t slot = rp.slot;
            const long long w0 = clock64();
            mbar_wait(bar(kBarFull + slot), rp.phase);
            vwait += clock64() - w0;
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < kVKeys / 16; ++kk) {
                const int key = kg * kVKeys + 16 * kk;  // key of the 256-key tile (P column)
                umma_bf16_pair(tmem + kTmemO + 128 * nh, dp + (uint64_t)((8192 * (key >> 6) + 2 * (key & 63)) >> 4),
                               dv + (uint64_t)((kSlotBytes * slot + 2048 * kk) >> 4), idesc_pv,
                               !(first && kg == 0 && kk == 0));
              }
              umma_commit_pair_mc(bar(kBarEmpty + slot), 3);
            }
            __syncwarp();
          }
        if (elect_one()) umma_commit_pair_mc(bar(kBarOFull + (gi & 1)), 3);
        __syncwarp();
        TRACE(5, gi);
        if (p.trace && cid == 0 && gi < 64 && lane == 0) p.trace[12 * 64 + gi] = vwait;
      };
      // the next unit is decoded before the last PV, whose wait for the last P would otherwise be followed
      // by ~1K cycles of index math with the tensor pipe idle
      Unit U = make_unit(p, unit_index(p, cid < n_iter_total ? cid : 0));
      for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
        const uint32_t g0 = g;
        for (int i = 0; i < U.n_tiles; ++i) {
          issue_s(g0 + i, i == 0, i == U.n_tiles - 1);
          if (i >= 1) issue_pv(g0 + i - 1, i - 1 == 0);
        }
        const int nt = U.n_tiles;
        if (it + ncl < n_iter_total) U = make_unit(p, unit_index(p, it + ncl));
        issue_pv(g0 + nt - 1, nt == 1);
        g += nt;
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
    constexpr bool calib = kCalib;
    const float alpha = calib ? *p.alpha : 0.f, om_alpha = 1.f - alpha;
    double gacc = 0.0;  // this thread's part of d_alpha (fused calibration with d_o_hat)
    bool read_pend = false;  // the last epilogue's second store round may still be reading the P buffer
    // units are decoded one ahead, inside the previous epilogue while a TMA store reads its staging
    Unit Un = make_unit(p, unit_index(p, cid < n_iter_total ? cid : 0));
    for (int64_t it = cid; it < n_iter_total; it += ncl, ++uc) {
      const Unit U = Un;
      const int64_t row_g = U.row0 + 64 * rank + r;
      const bool row_ok = row_g < rows_b;
      const int64_t row_c = row_ok ? row_g : rows_b - 1;
      const int64_t my_tok = p.q_start + (p.small ? (int64_t)p.div_heads.div((uint32_t)row_c) : row_c / p.heads);
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
#if MLA_SOFTMAX_V2
        float mx[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // 4 chains of 3-input max (FMNMX3) over v[4 k + c]
          mx[c] = fmax3(__uint_as_float(v[c]), __uint_as_float(v[4 + c]), __uint_as_float(v[8 + c]));
#pragma unroll
          for (int k = 3; k < 15; k += 2)
            mx[c] = fmax3(mx[c], __uint_as_float(v[4 * k + c]), __uint_as_float(v[4 * k + 4 + c]));
          mx[c] = fmaxf(mx[c], __uint_as_float(v[60 + c]));
        }
        float tmax = fmaxf(fmax3(mx[0], mx[1], mx[2]), mx[3]) * sl2;
#else
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
#endif
        float* rb = red + buf * 256;
        rb[q4 * 64 + r] = tmax;
        if (read_pend) {  // P is written after this barrier: the previous output store must have read it
          if (warp == 2 && lane == 0) bulk_wait_group_read0();
          read_pend = false;
        }
        named_bar_sync(1, kSmThreads);
        tmax = fmaxf(fmaxf(rb[r], rb[64 + r]), fmaxf(rb[128 + r], rb[192 + r]));
        const bool resc = tmax > m_used + 8.0f;
        const float m_new = resc ? tmax : m_used;
        const float corr = resc ? ex2(m_used - m_new) : 1.0f;
        // P = exp2(s * scale - m): 4 independent partial sums; packed to bf16 pairs
        uint32_t pk[32];
#if MLA_SOFTMAX_V2
        // scale-subtract and row sums on pairs (FFMA2 / FADD2): half the FP32 instructions of the scalar form
        float ps0, ps1, ps2 = 0.f, ps3 = 0.f;
        {
          const uint64_t sl2v = f2pack(sl2, sl2), nmv = f2pack(-m_new, -m_new);
          uint64_t acc0 = f2pack(0.f, 0.f), acc1 = acc0;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            float y0, y1;
            f2unpack(ffma2(f2pack(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])), sl2v, nmv), y0, y1);
            const float e0 = ex2(y0), e1 = ex2(y1);
            const uint64_t e = f2pack(e0, e1);
            if (j & 1)
              acc1 = fadd2(acc1, e);
            else
              acc0 = fadd2(acc0, e);
            pk[j] = pack_bf16x2(e0, e1);
          }
          f2unpack(fadd2(acc0, acc1), ps0, ps1);
        }
#else
        float ps0 = 0.f, ps1 = 0.f, ps2 = 0.f, ps3 = 0.f;
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
#endif
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
      // calibration with d_o_hat: the warp's 32 rows x 128 dims of d_o_hat are read coalesced (an instruction
      // covers 4 rows x 128 B: lanes 8 j .. 8 j + 7 one row's 64 dims) and transposed through the idle P buffer
      // (4 KB per warp) into this thread's row; the first 64 dims are requested before the wait for the last PV
      // (per-thread row reads touched 32 rows, i.e. 32 L1 wavefronts, per instruction)
      const int64_t rows_all = (int64_t)p.n_q * p.heads;
      const int64_t drow0 = U.row0 + 64 * rank + 32 * (wq & 1);  // the warp's first row
      const uint8_t* dbase = kDoHat
                                 ? p.d_o_hat + ((int64_t)U.bi * p.o_sb + 256 * (int)ch + 128 * (int)kh) * 2 + 16 * (lane & 7)
                                 : nullptr;
      const uint32_t dscr = sbase + kOffP + (warp - 2) * 4096;  // this warp's transpose scratch
      uint4 dl[8];
      auto dload_pair = [&](int pp) {  // dims 64 pp .. 64 pp + 63 of the warp's 128, rows drow0 + 4 i + lane / 8
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t rg = drow0 + 4 * i + (lane >> 3);
          dl[i] = dbase && rg < rows_all ? ldg_nc_v4(dbase + rg * kDv * 2 + 128 * pp) : make_uint4(0, 0, 0, 0);
        }
      };
      auto dstage = [&]() {  // row 4 i + lane / 8 of the scratch, 16-B unit lane % 8 (swizzled by row & 7)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t rl = 4 * i + (lane >> 3);
          st_shared_v4(dscr + rl * 128 + ((((uint32_t)lane & 7) ^ (rl & 7)) << 4), dl[i].x, dl[i].y, dl[i].z, dl[i].w);
        }
      };
      if constexpr (kDoHat) dload_pair(0);
      mbar_wait(bar(kBarOFull + (gl & 1)), (gl >> 1) & 1);
      tc_fence_after();
      if constexpr (kDoHat) {  // the P buffer is free: dims 0-63 into the scratch, then the loads of dims 64-127
        dstage();
        __syncwarp();
        dload_pair(1);
      }
      float* ls = red + ((gl + 1) & 1) * 256;  // the exchange buffer not used by the last tile
      ls[q4 * 64 + r] = lrow;
      named_bar_sync(1, kSmThreads);
      const float ltot = (ls[r] + ls[64 + r]) + (ls[128 + r] + ls[192 + r]);
      const float inv = 1.0f / ltot;
      named_bar_sync(1, kSmThreads);  // everyone has read ls before the next unit's first exchange writes red
      if (p.out_bf16) {
        // O (this thread: row r, dims 256 ch + 128 kh + [0, 128)) -> bf16 registers; O is then free for
        // the next unit's PV. Stores go out as TMA boxes [64 rows x 64 dims] staged in the P buffer (idle
        // between PV(T-1) and the next unit's first softmax): a flood of st.global from 256 threads queues
        // ahead of the MMA warp's mbarrier operations and stalls the tensor pipe at every unit boundary.
        uint32_t w[64];
        if constexpr (!calib) {
#pragma unroll
          for (int c = 0; c < 4; c += 2) {  // two TMEM loads per wait
            uint32_t ova[32], ovb[32];
            tmem_ld32(taddr + kTmemO + 128 * ch + 32 * c, ova);
            tmem_ld32(taddr + kTmemO + 128 * ch + 32 * (c + 1), ovb);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              w[16 * c + j] = pack_bf16x2(__uint_as_float(ova[2 * j]) * inv, __uint_as_float(ova[2 * j + 1]) * inv);
              w[16 * (c + 1) + j] = pack_bf16x2(__uint_as_float(ovb[2 * j]) * inv, __uint_as_float(ovb[2 * j + 1]) * inv);
            }
          }
        } else {
          // Eq. 3 on this thread's 128 outputs: o_hat = fma(alpha, O, (1 - alpha) O') with O' the fp32 SSA
          // result (alpha = 0 gives exactly the plain bf16 output, alpha = 1 gives O), and
          // d_alpha += d_o_hat (O - O'). O and d_o_hat are read straight from global (bf16, 64 B per chunk).
          float gs = 0.f;
          mbar_wait(bar(kBarOfFull), uc & 1);  // this unit's O_full rows, staged in the Q region
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld32(taddr + kTmemO + 128 * ch + 32 * c, ov);
            uint32_t xw[16], dw[16];
            if (kDoHat && c == 2) {  // every lane has read dims 0-63 of its row: dims 64-127 into the scratch
              __syncwarp();
              dstage();
              __syncwarp();
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // this row's 32 dims of chunk c: units 4 (c & 1) .. of its scratch row
              uint4 x4 = make_uint4(0, 0, 0, 0);
              if (kDoHat)
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(x4.x), "=r"(x4.y), "=r"(x4.z), "=r"(x4.w)
                             : "r"(dscr + (uint32_t)lane * 128 + ((((uint32_t)(4 * (c & 1) + q)) ^ ((uint32_t)lane & 7)) << 4)));
              dw[4 * q] = x4.x; dw[4 * q + 1] = x4.y; dw[4 * q + 2] = x4.z; dw[4 * q + 3] = x4.w;
            }
            // O_full box m = dims [64 m, +64): row r at m * 8192 + 128 r, 16-B units swizzled by r & 7
            const uint8_t* ofs = smem + kOffQ + of_slot(4 * ch + 2 * kh + (c >> 1)) * 8192 + r * 128;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 x4 = *reinterpret_cast<const uint4*>(ofs + ((((c & 1) * 4 + q) ^ (r & 7)) << 4));
              xw[4 * q] = x4.x; xw[4 * q + 1] = x4.y; xw[4 * q + 2] = x4.z; xw[4 * q + 3] = x4.w;
            }
            if (c & 1) {  // this warp is done with O_full box 4 ch + 2 kh + (c >> 1): its slot may take Q
              __syncwarp();
              if (lane == 0) mbar_arrive_local(bar(kBarOfEmpty + of_slot(4 * ch + 2 * kh + (c >> 1))));
            }
            tmem_wait_ld();
            uint32_t wc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float y0 = __uint_as_float(ov[2 * j]) * inv, y1 = __uint_as_float(ov[2 * j + 1]) * inv;
              const float x0 = bf_lo(xw[j]), x1 = bf_hi(xw[j]);
              wc[j] = pack_bf16x2(fmaf(alpha, x0, om_alpha * y0), fmaf(alpha, x1, om_alpha * y1));
              if constexpr (kDoHat) gs = fmaf(bf_lo(dw[j]), x0 - y0, fmaf(bf_hi(dw[j]), x1 - y1, gs));
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) w[16 * c + j] = wc[j];
          }
          gacc += (double)gs;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(ofree);
        if (warp == 2 && lane == 0) TRACE(17, gl);
        const uint32_t stage = sbase + kOffP;
        if constexpr (kDoHat) named_bar_sync(1, kSmThreads);  // every warp is done with its d_o_hat scratch
#pragma unroll
        for (int rd = 0; rd < 2; ++rd) {  // round rd: the warps with ch == rd, dims [256 rd, +256) = 4 boxes
          if (rd == 1) {  // round 0's store reads the staging: decode the next unit meanwhile, then wait
            if (it + ncl < n_iter_total) Un = make_unit(p, unit_index(p, it + ncl));
            if (warp == 2 && lane == 0) bulk_wait_group_read0();
            named_bar_sync(1, kSmThreads);
          }
          if (ch == (uint32_t)rd) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t box = stage + (2 * kh + (c >> 1)) * 8192 + r * 128;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t u = (c & 1) * 4 + q;
                st_shared_v4(box + ((u ^ (r & 7)) << 4), w[16 * c + 4 * q], w[16 * c + 4 * q + 1],
                             w[16 * c + 4 * q + 2], w[16 * c + 4 * q + 3]);
              }
            }
            fence_proxy_async_smem();
          }
          named_bar_sync(1, kSmThreads);
          if (warp == 2 && lane == 0) TRACE(18 + 2 * rd, gl);
          if (warp == 2 && lane == 0) {
            for (int m = 0; m < 4; ++m)
              tma_store_3d(&p.o_map, stage + m * 8192, 64 * (4 * rd + m), (int32_t)(U.row0 + 64 * rank), U.bi);
            bulk_commit_group();
          }
          if (warp == 2 && lane == 0) TRACE(19 + 2 * rd, gl);
        }
        read_pend = true;  // round 1's read is awaited before the next unit's first P write
      } else {
        char* obase = reinterpret_cast<char*>(p.o) + ((int64_t)U.bi * p.o_sb + (row_ok ? row_g : 0) * kDv) * 4;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t ov[32];
          tmem_ld32(taddr + kTmemO + 128 * ch + 32 * c, ov);
          tmem_wait_ld();
          const int dim0 = 256 * (int)ch + 128 * (int)kh + 32 * c;
          if (row_ok) {
            char* dst = obase + dim0 * 4;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              st_global_v4(dst + 16 * q, __float_as_uint(__uint_as_float(ov[4 * q]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 1]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 2]) * inv),
                           __float_as_uint(__uint_as_float(ov[4 * q + 3]) * inv));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(ofree);
        if (it + ncl < n_iter_total) Un = make_unit(p, unit_index(p, it + ncl));
      }
      if (p.lse && row_ok && q4 == 0) {
        const int64_t h = row_g % p.heads, tl_ = row_g / p.heads;
        p.lse[((int64_t)U.bi * p.heads + h) * p.lse_sh + tl_] = (m_used + __log2f(ltot)) * ln2;
      }
      g += U.n_tiles;
    }
    if (warp == 2 && lane == 0) bulk_wait_group0();  // output stores complete before exit
    if (kCalib && p.part) {  // d_alpha: fixed-order per-CTA fp64 partial (deterministic)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gacc += __shfl_xor_sync(0xffffffffu, gacc, o);
      named_bar_sync(1, kSmThreads);  // red[] is free: every unit's exchanges are done
      double* wsum = reinterpret_cast<double*>(red);
      if (lane == 0) wsum[warp - 2] = gacc;
      named_bar_sync(1, kSmThreads);
      if (threadIdx.x == 64) {
        double t = 0.0;
        for (int i = 0; i < (int)kSoftmaxWarps; ++i) t += wsum[i];
        p.part[blockIdx.x] = t;
      }
    }
    if (kCalib && p.status && blockIdx.x == 0 && threadIdx.x == 64)
      *p.status = (alpha >= 0.f && alpha <= 1.f) ? LOZA_OK : LOZA_ERR_INVALID;
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
  p.lse_sh = a.lse_sh;
  if (a.calib) {
    if (!encode_3d(&p.of_map, a.calib->o_full, kDv, (uint64_t)a.n_q * a.heads, a.batch, kDv, a.o_sb, 64))
      return cudaErrorInvalidValue;
    p.o_full = reinterpret_cast<const uint8_t*>(a.calib->o_full);
    p.d_o_hat = reinterpret_cast<const uint8_t*>(a.calib->d_o_hat);
    p.alpha = a.calib->alpha;
    p.part = a.calib->part;
    p.status = a.calib->status;
  }
  const int64_t rows = (int64_t)a.n_q * a.heads;
  p.units_per_batch = (rows + 127) / 128;
  p.trace = g_debug_trace;
  p.total_units = p.units_per_batch * a.batch;
  if (p.total_units == 0) return cudaSuccess;
  const int64_t lim = (int64_t)1 << 31;
  p.small = p.total_units * 128 < lim && rows + 128 < lim && a.q_start + a.n_q + 128 < lim && a.n_kv + 128 < lim;
  if (p.small) {
    p.div_upb.init((uint32_t)p.units_per_batch);
    p.div_heads.init((uint32_t)a.heads);
    p.div_b.init((uint32_t)(a.sparse ? a.b : 128));
  }
  if (!encode_3d(&p.q_map, a.q, kDqk, rows, a.batch, kDqk, a.q_sb, 64)) return cudaErrorInvalidValue;
  if (a.out_bf16 && !encode_3d(&p.o_map, a.o, kDv, rows, a.batch, kDv, a.o_sb, 64)) return cudaErrorInvalidValue;
  p.nseg = a.kv.nseg;
  for (int i = 0; i < a.kv.nseg; ++i) {
    const KvSeg& s = a.kv.seg[i];
    p.seg_begin[i] = s.pos_begin;
    const uint64_t len = (uint64_t)(s.pos_end - s.pos_begin);
    p.seg_len[i] = (int32_t)len;
    if (!encode_3d(&p.k_map[i], s.k, kDqk, len, a.batch, s.k_st, s.k_sb, 128)) return cudaErrorInvalidValue;
    if (!encode_4d_chunks(&p.k2_map[i], s.k, kDqk, len, a.batch, s.k_st, s.k_sb, 128, 2)) return cudaErrorInvalidValue;
    if (!encode_4d_chunks(&p.v_map[i], s.v, kDv, len, a.batch, s.v_st, s.v_sb, kVKeys, 2)) return cudaErrorInvalidValue;
  }
  {  // per launch (the attribute is per device; a process may drive several GPUs)
    const int mode = a.calib ? (a.calib->d_o_hat ? 2 : 1) : 0;
    cudaError_t e = mode == 2   ? cudaFuncSetAttribute(prefill_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       kSmemAlloc)
                    : mode == 1 ? cudaFuncSetAttribute(prefill_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       kSmemAlloc)
                                : cudaFuncSetAttribute(prefill_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       kSmemAlloc);
    if (e != cudaSuccess) return e;
  }
  const int sms = device_sm_count();
  int64_t ncl = sms / 2;
  if (ncl > p.total_units) ncl = p.total_units;
  if (a.calib && a.calib->d_o_hat)
    prefill_tc_kernel<2><<<(unsigned)(2 * ncl), kThreads, kSmemAlloc, st>>>(p);
  else if (a.calib)
    prefill_tc_kernel<1><<<(unsigned)(2 * ncl), kThreads, kSmemAlloc, st>>>(p);
  else
    prefill_tc_kernel<0><<<(unsigned)(2 * ncl), kThreads, kSmemAlloc, st>>>(p);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && a.calib && a.calib->part)
    e = launch_dalpha_reduce(a.calib->part, (int)(2 * ncl), a.calib->alpha, a.calib->d_alpha, st);
  return e;
}

}  // namespace loza

// debug hook (not part of include/loza.h): record a clock64 timeline of cluster 0 into dev_ptr[17*64]
extern "C" void loza_debug_set_trace(void* dev_ptr) { loza::g_debug_trace = (unsigned long long*)dev_ptr; }
