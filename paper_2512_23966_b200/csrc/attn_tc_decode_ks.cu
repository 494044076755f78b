// SSA decode, key-split CTA pair (Eq. 4 at p = seq_len - 1).
//
// One cluster of two CTAs per sequence; each CTA owns every other 64-key item of the sequence's selected
// window (sink block(s) + the last l blocks) and runs its own online softmax over them -- no per-item
// dependency between the two CTAs. The partials are merged once at the end through distributed shared
// memory: CTA r finalises output dims [256 r, 256 r + 256).
//
//  * An item = 64 keys x 576 dims, one 72 KB TMA box ([9 chunks][64 keys][64 dims], SWIZZLE_128B). The
//    same SMEM tile is the A operand of S^T = K Q^T (K-major, M = 64 keys) and, read MN-major, of
//    O^T += V^T P (V = its first 512 dims): the latent window is read from HBM once and staged once.
//    Two ring slots (144 KB) + Q (72 KB, all 64 heads) fill the SMEM.
//  * S^T: 36 UMMAs M64 N64 K16 (cta_group::1) into TMEM (M=64 layout: keys 16 q .. 16 q + 15 on lanes
//    32 q .. 32 q + 15), double-buffered. P (bf16 [64 keys][64 heads], the MN-major B operand of PV) is
//    written over the item's RoPE chunk, which S^T(i) has finished reading when its commit fires.
//  * O^T: 4 groups of M128 (dims) x N64 (heads) fp32 = 256 TMEM columns; PV = 16 UMMAs M128 N64 K16.
//  * Softmax with a lazily updated max: each (key, head) logit x is compared with the running m_h; only
//    when some x exceeds m_h + kLazy anywhere in the CTA (one barrier.red.or per item; always on the
//    CTA's first item) does the CTA take the exact path (per-head item max through shared memory,
//    rescale of O^T and of the partial sums). Otherwise P = 2^(x - m_h) straight away: no cross-thread
//    reduction on the common path. Any m_h <= the running max is exact for the softmax (the shift cancels),
//    and x - m_h <= kLazy keeps P and the sums far from overflow.
//  * Merge: per-head (m, l) swapped through DSMEM; each CTA scales its partial O^T of the partner's dims
//    by its weight 2^(m_r - M) / L and stores it into the partner's (idle) ring; the partner adds it to
//    its own scaled half, converts and TMA-stores. LSE = M + log2 L (natural log on output).
//  * Warp 0: TMA (Q once, then items in order); warp 1: UMMA issuer (S(i+1) before PV(i)); warps 2-9:
//    softmax (TMEM lane quarter q = warp % 4, heads 32 hh .. with hh = (warp - 2) / 4), merge, epilogue.
//  * Heads H < 64 (head-sharded decode): Q rows >= H are TMA zero-fill, their outputs are not stored.
#include <math.h>
#include <string.h>

#include "internal.h"
#include "sm100.cuh"

namespace loza {

namespace {
using namespace sm100;

constexpr int kDqk = 576, kDv = 512, kChunks = 9, kH = 64;
constexpr int kItemKeys = 64;
constexpr int kChunkBytes = kItemKeys * 128;       // [64 keys][64 dims] bf16
constexpr int kItemBytes = kChunks * kChunkBytes;  // 73728
constexpr int kQBytes = kChunks * kH * 128;        // 73728
constexpr int kSlots = 2;
constexpr int kThreads = 320;
constexpr float kLazy = 20.0f;  // log2 units: P <= 2^20 between exact updates

constexpr int kOffQ = 0;
constexpr int kOffRing = kOffQ + kQBytes;
constexpr int kOffBar = kOffRing + kSlots * kItemBytes;
constexpr int kBarFull = 0;                 // [2] ring slot loaded
constexpr int kBarEmpty = kBarFull + 2;     // [2] ring slot free (PV of its item done)
constexpr int kBarQFull = kBarEmpty + 2;
constexpr int kBarSFull = kBarQFull + 1;    // [2]
constexpr int kBarSFree = kBarSFull + 2;    // [2]
constexpr int kBarPFull = kBarSFree + 2;    // [2]
constexpr int kBarOFull = kBarPFull + 2;    // [2] PV(i) done
constexpr int kBarXch = kBarOFull + 2;      // [2] the partner's 32 KB group gi landed (bulk DSMEM copy)
constexpr int kNumBars = kBarXch + 2;
constexpr int kOffTmemPtr = kOffBar + kNumBars * 8;
constexpr int kOffRed = (kOffTmemPtr + 4 + 15) & ~15;  // float [4 quarters][64 heads]
constexpr int kOffML = kOffRed + 4 * 64 * 4;            // float own m[64], own l[64], partner m[64], partner l[64]
constexpr int kOffMs = kOffML + 4 * 64 * 4;             // float running max m_h [64], rescale factors [64]
constexpr int kOffW = kOffMs + 2 * 64 * 4;              // float merge weight of this CTA's half per head [64]
constexpr int kSmemUsed = kOffW + 64 * 4;
constexpr int kSmemAlloc = kSmemUsed;
static_assert(kSmemAlloc <= 232448, "smem");
constexpr int kXchBytes = 2 * 64 * 128 * 4;           // fp32 [2 groups][64 heads][128 dims]
constexpr int kXchGroupBytes = kXchBytes / 2;
constexpr int kOffXch = kOffRing;                      // merge: the partner's scaled half of this CTA's dims
constexpr int kOffStage = kOffRing + kXchBytes;        // merge: this CTA's scaled half of the partner's dims
constexpr int kOffOut = kOffQ;     // bf16 output staging: 4 boxes [64 heads][64 dims] (32 KB)

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kTmemO = 0, kTmemS = 256;  // O^T group g at 64 g; S^T buffer b at 256 + 64 b
constexpr uint32_t kSmThreads = 256;

struct KsParams {
  CUtensorMap q_map, k_map, o_map;  // k_map: 4-D {64, rows, 9 chunks, batch}, box {64, 64 keys, 9, 1}
  const int32_t* seq_lens;
  int32_t batch, heads, s, l, b;
  int32_t ring;
  int64_t t_cap;
  int32_t n_rows;       // cache rows; an absent item maps here (out of bounds, zero-filled)
  const uint8_t* kraw;  // contiguous cache rows (L2 prefetch before the dependency wait), or NULL
  const uint8_t* qraw;
  int64_t k_sb_bytes, k_st_bytes, q_sb_bytes, q_sh_bytes;
  float scale_log2;
  void* o;
  int64_t o_sb, o_sh;
  int32_t out_bf16;
  float* lse;
  int32_t* status;  // nullable: LOZA_ERR_SHAPE when a seq_len was outside [1, t_cap] (clamped)
  unsigned long long* trace;  // debug timeline of cluster 0 (NULL in production): [slot][rank][32]
};

#define KTRACE(slot, idx)                                                                          \
  do {                                                                                             \
    if (p.trace && blockIdx.x < 2 && (idx) < 32 && (threadIdx.x & 31) == 0)                        \
      p.trace[((slot) * 2 + (blockIdx.x & 1)) * 32 + (idx)] = clock64();                          \
  } while (0)

struct Window {
  int32_t pos;                         // query position seq_len - 1
  int32_t n_sink, loc_begin, n_sub;    // selected 128-key sub-blocks: sinks [0, n_sink), locals from loc_begin
  int32_t n_items;                     // 64-key items holding at least one key <= pos
};
__device__ __forceinline__ Window window(const KsParams& p, int bi, bool* clamped) {
  int64_t L = p.seq_lens[bi];
  *clamped = L < 1 || L > p.t_cap;
  L = L < 1 ? 1 : (L > p.t_cap ? p.t_cap : L);
  Window w;
  w.pos = (int32_t)(L - 1);
  const int32_t last = w.pos >> 7, tpb = p.b >> 7, QB = w.pos / p.b;
  int32_t sink_end = (QB + 1 < p.s ? QB + 1 : p.s) * tpb;
  if (sink_end > last + 1) sink_end = last + 1;
  int32_t lb = QB - p.l + 1;
  if (lb < p.s) lb = p.s;
  lb *= tpb;
  int32_t le = (QB + 1) * tpb;
  if (le > last + 1) le = last + 1;
  w.n_sink = sink_end;
  w.loc_begin = lb;
  w.n_sub = sink_end + (le > lb ? le - lb : 0);
  // the last selected sub-block holds pos: its second half is an item only if pos reaches it
  w.n_items = 2 * (w.n_sub - 1) + ((w.pos & 127) >= 64 ? 2 : 1);
  return w;
}
// absolute first key of item j (j < n_items)
__device__ __forceinline__ int32_t item_k0(const Window& w, int j) {
  const int sub = j >> 1;
  return (sub < w.n_sink ? sub : w.loc_begin + (sub - w.n_sink)) * 128 + 64 * (j & 1);
}
// cache row of key k0: identity, or the bounded ring's slot of its block (ring_cache.cu)
__device__ __forceinline__ int32_t kv_row(const KsParams& p, int32_t k0) {
  if (!p.ring) return k0;
  const int32_t kb = k0 / p.b;
  if (kb < p.s) return k0;
  return p.s * p.b + ((kb - p.s) % p.l) * p.b + (k0 - kb * p.b);
}
__device__ __forceinline__ bool bar_red_or(uint32_t id, uint32_t n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred pi, po;\n\t"
      "setp.ne.u32 pi, %1, 0;\n\t"
      "barrier.cta.red.or.pred po, %2, %3, pi;\n\t"
      "selp.u32 %0, 1, 0, po;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}
// 16 TMEM lanes x 32 columns (16x256b.x4): thread i gets lanes (i/4, i/4 + 8) x columns 8k + 2 (i%4) + {0, 1}
// as r[4k + {0, 1}] (lane i/4) and r[4k + {2, 3}] (lane i/4 + 8), k = 0..3
__device__ __forceinline__ void tmem_ld16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void bulk_copy_to_cluster(uint32_t dst_cluster, uint32_t src, uint32_t bytes,
                                                     uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst_cluster),
      "r"(src), "r"(bytes), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void st_shared_b32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(2, 1, 1)
    decode_ks_kernel(const __grid_constant__ KsParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int i) { return bar0 + 8u * (uint32_t)i; };
  uint32_t* tmem_ptr_smem = reinterpret_cast<uint32_t*>(smem + kOffTmemPtr);
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  float* ml = reinterpret_cast<float*>(smem + kOffML);
  float* ms = reinterpret_cast<float*>(smem + kOffMs);  // running max per head (same for every softmax thread)
  const uint32_t rank = cluster_ctarank(), partner = rank ^ 1;
  const int bi = (int)(blockIdx.x >> 1);

  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 2) KTRACE(0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kNumBars; ++i) mbar_init(bar(i), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(kBarSFree + i), kSmThreads / 32);
      mbar_init(bar(kBarPFull + i), kSmThreads / 32);
    }
    fence_mbar_init();
    // armed long before the partner's bulk copy can complete on it (after the first cluster barrier)
    mbar_arrive_expect_tx(bar(kBarXch), kXchGroupBytes);
    mbar_arrive_expect_tx(bar(kBarXch + 1), kXchGroupBytes);
    prefetch_tmap(&p.q_map);
    prefetch_tmap(&p.k_map);
  }
  if (warp == 1) tmem_alloc<1>(smem_u32(tmem_ptr_smem), kTmemCols);
  if (threadIdx.x < 64) ms[threadIdx.x] = -INFINITY;
  // Under programmatic dependent launch this CTA may start while the previous kernel still runs: pull Q
  // and the first item into L2 before waiting for it (hints only; seq_lens may be stale here).
  if (warp == 0 && lane == 0 && p.kraw) {
    bool c;
    const Window w0 = window(p, bi, &c);
    if ((int)rank < w0.n_items) {
      const int32_t row = kv_row(p, item_k0(w0, (int)rank));
      if (row + kItemKeys <= p.n_rows)
        bulk_prefetch_l2(p.kraw + bi * p.k_sb_bytes + row * p.k_st_bytes, (uint32_t)(kItemKeys * p.k_st_bytes));
    }
    if (p.qraw) bulk_prefetch_l2(p.qraw + bi * p.q_sb_bytes, (uint32_t)(p.heads * p.q_sh_bytes));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_smem;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // inputs of the previous kernel are visible from here
  if (warp == 2) KTRACE(0, 1);

  bool clamped;
  const Window w = window(p, bi, &clamped);
  const int n_my = (w.n_items - (int)rank + 1) / 2;  // items rank, rank + 2, ...
  if (clamped && p.status && rank == 0 && threadIdx.x == 0) atomicExch(p.status, (int32_t)LOZA_ERR_SHAPE);

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    const uint64_t pol_q = policy_evict_first(), pol_kv = policy_evict_first();
    if (elect_one()) {
      // one 72 KB box per item: whole 1152-B cache rows (DRAM page locality; per-chunk boxes measured ~2x slower)
      mbar_arrive_expect_tx(bar(kBarQFull), kQBytes);
      for (int c = 0; c < kChunks; ++c)
        tma_load_3d(sbase + kOffQ + c * (kH * 128), &p.q_map, 64 * c, 0, bi, bar(kBarQFull), pol_q);
      for (int t = 0; t < n_my; ++t) {
        const int slot = t & 1;
        if (t >= kSlots) mbar_wait(bar(kBarEmpty + slot), ((t >> 1) - 1) & 1);
        KTRACE(1, t);
        const int32_t row = kv_row(p, item_k0(w, (int)rank + 2 * t));
        mbar_arrive_expect_tx(bar(kBarFull + slot), kItemBytes);
        tma_load_4d(sbase + kOffRing + slot * kItemBytes, &p.k_map, 0, row, 0, bi, bar(kBarFull + slot), pol_kv);
        if (p.kraw && t + kSlots < n_my) {
          // Two items in SMEM are ~144 KB in flight per SM, too few to cover the HBM latency under load: keep
          // the item after next on its way into L2, so the load that waits for a free slot hits L2.
          const int32_t r2 = kv_row(p, item_k0(w, (int)rank + 2 * (t + kSlots)));
          if (r2 + kItemKeys <= p.n_rows)
            bulk_prefetch_l2(p.kraw + bi * p.k_sb_bytes + (int64_t)r2 * p.k_st_bytes,
                             (uint32_t)(kItemKeys * p.k_st_bytes));
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------------ UMMA issuer
    constexpr uint32_t idesc_s = idesc_bf16_f32(64, 64, false, false);
    constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 64, true, true);
    const uint64_t dq = sdesc_sw128(sbase + kOffQ, 16, 1024);
    const uint64_t dk = sdesc_sw128(sbase + kOffRing, 16, 1024);
    const uint64_t dv = sdesc_sw128(sbase + kOffRing, kChunkBytes, 1024);  // V^T: M = dims over 2 chunks
    const uint64_t dp = sdesc_sw128(sbase + kOffRing + 8 * kChunkBytes, kChunkBytes, 1024);  // P in chunk 8
    auto issue_pv = [&](int t) {
      const int slot = t & 1, buf = t & 1;
      KTRACE(3, t);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_1sm(tmem + kTmemO + 64 * g,
                          dv + (uint64_t)((slot * kItemBytes + 2 * g * kChunkBytes + 2048 * kk) >> 4),
                          dp + (uint64_t)((slot * kItemBytes + 2048 * kk) >> 4), idesc_pv, (t | kk) != 0);
        umma_commit_1sm(bar(kBarEmpty + slot));
        umma_commit_1sm(bar(kBarOFull + buf));
      }
      __syncwarp();
    };
    // Event loop: S^T(ns) as soon as item ns landed (and S buffer ns & 1 is free), PV(np) as soon as P(np) is
    // written -- neither waits behind the other's barrier (a PV held back by a late load would hold the ring
    // slot of the load after next).
    if (n_my > 0) mbar_wait(bar(kBarQFull), 0);
    int ns = 0, np = 0;
    while (np < n_my) {
      if (ns < n_my && mbar_test(bar(kBarFull + (ns & 1)), (ns >> 1) & 1) &&
          (ns < 2 || mbar_test(bar(kBarSFree + (ns & 1)), ((ns >> 1) - 1) & 1))) {
        const int slot = ns & 1, buf = ns & 1;
        KTRACE(2, ns);
        tc_fence_after();
        if (elect_one()) {
          for (int c = 0; c < kChunks; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16_1sm(tmem + kTmemS + 64 * buf,
                            dk + (uint64_t)((slot * kItemBytes + c * kChunkBytes + 32 * k) >> 4),
                            dq + (uint64_t)((c * (kH * 128) + 32 * k) >> 4), idesc_s, (c | k) != 0);
          umma_commit_1sm(bar(kBarSFull + buf));
        }
        __syncwarp();
        ++ns;
      }
      if (np < ns && mbar_test(bar(kBarPFull + (np & 1)), (np >> 1) & 1)) {
        issue_pv(np);
        ++np;
      }
    }
  } else {
    // ------------------------------------------------------------------ softmax (warps 2..9)
    // warp (q, hh): keys 16 q .. 16 q + 15 of the item (TMEM lanes 32 q ..), heads 32 hh .. 32 hh + 31. Thread
    // i holds keys kA = 16 q + i/4 and kB = kA + 8, heads h(k, e) = 32 hh + 8 k + 2 (i%4) + e (jj = 2 k + e).
    const uint32_t q = warp & 3, hh = (warp - 2) >> 2;
    const uint32_t t0 = lane & 3, t1 = lane >> 2;
    const uint32_t kA = 16 * q + t1, kB = kA + 8;
    const uint32_t taddr = tmem + ((32 * q) << 16);
    const float sl2 = p.scale_log2;
    float* corr_s = ms + 64;
    float m[8], l[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      m[jj] = -INFINITY;
      l[jj] = 0.f;
    }
    auto head = [&](int jj) -> uint32_t { return 32 * hh + 8 * (jj >> 1) + 2 * t0 + (jj & 1); };
    for (int t = 0; t < n_my; ++t) {
      const int slot = t & 1, buf = t & 1;
      const int32_t k0 = item_k0(w, (int)rank + 2 * t);
      const bool vA = k0 + (int32_t)kA <= w.pos, vB = k0 + (int32_t)kB <= w.pos;
      mbar_wait(bar(kBarSFull + buf), (t >> 1) & 1);
      if (warp == 2) KTRACE(4, t);
      tc_fence_after();
      uint32_t v[16];
      tmem_ld16x256b_x4(taddr + kTmemS + 64 * buf + 32 * hh, v);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarSFree + buf));
      float xa[8], xb[8];
      bool viol = false;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int k = jj >> 1, e = jj & 1;
        xa[jj] = vA ? __uint_as_float(v[4 * k + e]) * sl2 : -INFINITY;
        xb[jj] = vB ? __uint_as_float(v[4 * k + 2 + e]) * sl2 : -INFINITY;
        viol |= fmaxf(xa[jj], xb[jj]) > m[jj] + kLazy;
      }
      const bool exact = bar_red_or(2, kSmThreads, viol);
      if (warp == 2) KTRACE(5, t);
      if (exact) {
        if (warp == 2) KTRACE(6, t);
        // exact path: per-head max of this item, m = max(m, item max); rescale l and O^T
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          float r = fmaxf(xa[jj], xb[jj]);
          r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, 4));
          r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, 8));
          r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, 16));
          if (t1 == 0) red[q * 64 + head(jj)] = r;
        }
        named_bar_sync(1, kSmThreads);
        bool moved = false;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const uint32_t h = head(jj);
          const float hm = fmaxf(fmaxf(red[h], red[64 + h]), fmaxf(red[128 + h], red[192 + h]));
          const float mn = fmaxf(m[jj], hm);
          const float c = m[jj] == -INFINITY ? 0.f : ex2(m[jj] - mn);
          moved |= mn != m[jj];
          l[jj] *= c;
          m[jj] = mn;
          if (q == 0 && t1 == 0) {
            corr_s[h] = c;
            ms[h] = mn;
          }
        }
        moved = bar_red_or(3, kSmThreads, moved);  // also orders corr_s before its reads
        if (t > 0 && moved) {  // O^T columns of this warp's 32 heads (lanes = dims), once PV(t-1) landed
          mbar_wait(bar(kBarOFull + ((t - 1) & 1)), ((t - 1) >> 1) & 1);
          tc_fence_after();
          const uint32_t t32 = tmem + ((32 * q) << 16);
#pragma unroll 1
          for (int g = 0; g < 4; ++g) {
            uint32_t ov[32];
            tmem_ld32(t32 + kTmemO + 64 * g + 32 * hh, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] = __float_as_uint(__uint_as_float(ov[j]) * corr_s[32 * hh + j]);
            tmem_st32(t32 + kTmemO + 64 * g + 32 * hh, ov);
          }
          tmem_wait_st();
          tc_fence_before();
        }
      }
      // P rows kA, kB: heads 32 hh + 8 k + 2 t0 + {0, 1} = 32-bit word t0 of 16-B unit 4 hh + k (SWIZZLE_128B)
      const uint32_t pbase = sbase + kOffRing + slot * kItemBytes + 8 * kChunkBytes;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a0 = ex2(xa[2 * k] - m[2 * k]), a1 = ex2(xa[2 * k + 1] - m[2 * k + 1]);
        const float b0 = ex2(xb[2 * k] - m[2 * k]), b1 = ex2(xb[2 * k + 1] - m[2 * k + 1]);
        l[2 * k] += a0 + b0;
        l[2 * k + 1] += a1 + b1;
        st_shared_b32(pbase + kA * 128 + (((4 * hh + k) ^ (kA & 7)) << 4) + 4 * t0, pack_bf16x2(a0, a1));
        st_shared_b32(pbase + kB * 128 + (((4 * hh + k) ^ (kB & 7)) << 4) + 4 * t0, pack_bf16x2(b0, b1));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_local(bar(kBarPFull + buf));
      if (warp == 2) KTRACE(7, t);
    }

    // ------------------------------------------------------------------ merge of the two key halves
    if (n_my > 0) {
      mbar_wait(bar(kBarOFull + ((n_my - 1) & 1)), ((n_my - 1) >> 1) & 1);
      tc_fence_after();
    }
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {  // over the 8 lanes sharing a head column (the warp's 16 keys)
      float r = l[jj];
      r += __shfl_xor_sync(0xffffffffu, r, 4);
      r += __shfl_xor_sync(0xffffffffu, r, 8);
      r += __shfl_xor_sync(0xffffffffu, r, 16);
      if (t1 == 0) red[q * 64 + head(jj)] = r;
    }
    named_bar_sync(1, kSmThreads);
    if (q == 2) {  // warps 2 and 6: own (m, l) of heads 32 hh .. to this CTA and to the partner
      const uint32_t h = 32 * hh + lane;
      const float lt = (red[h] + red[64 + h]) + (red[128 + h] + red[192 + h]);
      const float mt = ms[h];
      ml[h] = mt;
      ml[64 + h] = lt;
      st_cluster_f32(mapa(sbase + kOffML + (128 + h) * 4, partner), mt);
      st_cluster_f32(mapa(sbase + kOffML + (192 + h) * 4, partner), lt);
    }
  }
  // every CTA's items are done (its ring is idle) and (m, l) of both halves are in place
  if (warp == 2) KTRACE(8, 0);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) KTRACE(8, 1);
  if (warp >= 2) {
    const uint32_t q = warp & 3, hh = (warp - 2) >> 2;
    const uint32_t taddr = tmem + ((32 * q) << 16);
    float* wo = reinterpret_cast<float*>(smem + kOffW);
    const uint32_t tid = threadIdx.x - 64;
    if (tid < 64) {  // per head: this CTA's weight 2^(m_own - M) / L and (CTA 0) the LSE
      const float mo = ml[tid], lo = ml[64 + tid], mp = ml[128 + tid], lp = ml[192 + tid];
      const float M = fmaxf(mo, mp);
      const float ao = lo > 0.f ? ex2(mo - M) : 0.f, ap = lp > 0.f ? ex2(mp - M) : 0.f;
      const float L = ao * lo + ap * lp;
      wo[tid] = ao / L;
      if (rank == 0 && p.lse && tid < (uint32_t)p.heads)
        p.lse[(int64_t)bi * p.heads + tid] = (M + __log2f(L)) * 0.69314718055994531f;
    }
    named_bar_sync(1, kSmThreads);
    // the partner's dims (O^T groups 2 partner + gi), scaled, staged as fp32 [gi][64 heads][128 dims] (a warp's
    // 32 lanes = dims write 128 contiguous bytes) and sent group by group, one 32 KB bulk DSMEM copy each: the
    // second group's staging overlaps the first copy, the first group's combine the second copy
    float* stage = reinterpret_cast<float*>(smem + kOffStage);
#pragma unroll 1
    for (int gi = 0; gi < 2; ++gi) {
      uint32_t ov[32];
      if (n_my > 0) {
        tmem_ld32(taddr + kTmemO + 64 * (2 * partner + gi) + 32 * hh, ov);
        tmem_wait_ld();
      }
      float* dst = stage + (gi * 64 + 32 * hh) * 128 + 32 * q + lane;
#pragma unroll
      for (int j = 0; j < 32; ++j) dst[j * 128] = n_my > 0 ? __uint_as_float(ov[j]) * wo[32 * hh + j] : 0.f;
      fence_proxy_async_smem();
      named_bar_sync(1, kSmThreads);
      if (warp == 2 && lane == 0) {
        bulk_copy_to_cluster(mapa(sbase + kOffXch + gi * kXchGroupBytes, partner),
                             sbase + kOffStage + gi * kXchGroupBytes, kXchGroupBytes,
                             mapa(bar(kBarXch + gi), partner));
        bulk_commit_group();
      }
    }
    if (warp == 2) KTRACE(8, 2);
    float* ob = reinterpret_cast<float*>(p.o) + (int64_t)bi * p.o_sb + 256 * rank;  // fp32 output only
#pragma unroll 1
    for (int gi = 0; gi < 2; ++gi) {
      uint32_t ov[32];
      if (n_my > 0) {
        tmem_ld32(taddr + kTmemO + 64 * (2 * rank + gi) + 32 * hh, ov);
        tmem_wait_ld();
      }
      // the partner's copy completes on this CTA's barrier: spin (a suspended try_wait is not reliably woken
      // by a remote complete_tx; see attn_tc_decode_coop.cu)
      while (!mbar_test(bar(kBarXch + gi), 0)) {
      }
      if (warp == 2) KTRACE(8, 3 + gi);
      const uint32_t dl = 128 * gi + 32 * q + lane;  // dim within this CTA's 256
      const float* xr = reinterpret_cast<const float*>(smem + kOffXch) + (gi * 64 + 32 * hh) * 128 + 32 * q + lane;
      const uint32_t box = sbase + kOffOut + (dl >> 6) * 8192, col = dl & 63;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t h = 32 * hh + j;
        const float val = (n_my > 0 ? __uint_as_float(ov[j]) * wo[h] : 0.f) + xr[j * 128];
        if (p.out_bf16) {
          const uint32_t a = box + h * 128 + (((col >> 3) ^ (h & 7)) << 4) + (col & 7) * 2;
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)(pack_bf16x2(val, 0.f) & 0xFFFFu)));
        } else if (h < (uint32_t)p.heads) {
          ob[(int64_t)h * p.o_sh + dl] = val;
        }
      }
    }
    if (p.out_bf16) {
      fence_proxy_async_smem();
      named_bar_sync(1, kSmThreads);
      if (warp == 2 && lane == 0)
        for (int mm = 0; mm < 4; ++mm)
          tma_store_3d(&p.o_map, sbase + kOffOut + mm * 8192, 256 * (int)rank + 64 * mm, 0, bi);
    }
    if (warp == 2 && lane == 0) {  // the DSMEM copy's and the output store's reads of this CTA's smem are done
      bulk_commit_group();
      bulk_wait_group_read0();
    }
  }
  // No closing cluster barrier: the partner's last access to this CTA's shared memory is its bulk copy, which
  // completed before the spin above; this CTA's copies were read out (wait_group.read) and the partner waits
  // for their completion before it exits.
  if (warp == 2) KTRACE(8, 5);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, kTmemCols);
  }
}

}  // namespace

unsigned long long* g_ks_trace = nullptr;

bool decode_ks_eligible(const AttnProblem& a, int sms) {
  return a.sparse && a.heads >= 1 && a.heads <= kH && a.d_qk == kDqk && a.d_v == kDv && a.b % 128 == 0 &&
         2 * (int64_t)a.batch <= sms && a.n_kv < (1ll << 31);
}

cudaError_t launch_decode_ks(const AttnProblem& a, int32_t* status, cudaStream_t st) {
  if (a.heads < 1 || a.heads > kH || a.d_qk != kDqk || a.d_v != kDv) return cudaErrorNotSupported;
  if (a.n_kv >= (1ll << 31)) return cudaErrorNotSupported;
  KsParams p;
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
  const KvSeg& s = a.kv.seg[0];
  if (s.k_st == kDqk && s.v == s.k) {
    p.kraw = reinterpret_cast<const uint8_t*>(s.k);
    p.k_sb_bytes = s.k_sb * 2;
    p.k_st_bytes = s.k_st * 2;
  }
  if (a.q_sh == kDqk) {
    p.qraw = reinterpret_cast<const uint8_t*>(a.q);
    p.q_sb_bytes = a.q_sb * 2;
    p.q_sh_bytes = a.q_sh * 2;
  }
  p.scale_log2 = a.scale * 1.4426950408889634f;
  p.o = a.o;
  p.o_sb = a.o_sb;
  p.o_sh = a.o_sh;
  p.out_bf16 = a.out_bf16;
  p.lse = a.lse;
  p.status = status;
  p.trace = g_ks_trace;
  // V must be the first 512 columns of the KV rows (absorbed MLA): the item tile serves both roles
  if (s.v != s.k || s.v_st != s.k_st || s.v_sb != s.k_sb) return cudaErrorNotSupported;
  if (!encode_3d(&p.q_map, a.q, kDqk, (uint64_t)a.heads, a.batch, a.q_sh, a.q_sb, kH)) return cudaErrorInvalidValue;
  if (!encode_4d_chunks(&p.k_map, s.k, kDqk, (uint64_t)a.n_kv, a.batch, s.k_st, s.k_sb, kItemKeys, kChunks))
    return cudaErrorInvalidValue;
  if (a.out_bf16 && !encode_3d(&p.o_map, a.o, kDv, (uint64_t)a.heads, a.batch, a.o_sh, a.o_sb, kH))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(decode_ks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemAlloc);
  if (e != cudaSuccess) return e;
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
  e = cudaLaunchKernelEx(&cfg, decode_ks_kernel, p);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza

// debug hook (not part of include/loza.h): clock64 timeline of cluster 0 into dev_ptr[9 * 2 * 32]
extern "C" void loza_debug_set_ks_trace(void* dev_ptr) { loza::g_ks_trace = (unsigned long long*)dev_ptr; }
