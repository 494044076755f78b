// Bounded SSA KV cache: per sequence R = (s + l) * b rows,
// the s sink blocks at rows [0, s*b) and a ring of the l most recent blocks, block kb >= s at rows
// s*b + ((kb - s) mod l) * b. Appending rows in position order overwrites a ring slot exactly when a new
// block opens, i.e. the block-boundary eviction of SPEC.md:397 ("a local block expires when qb - kb >= l
// and kb >= s"), so the cache always holds {j : allowed(t, j)} for the next query t.
//
// Append of m rows at absolute positions pos0 .. pos0 + m - 1 (pos0 = the sequence's length before the
// append, from the device): only rows that survive the whole append are written (sink rows, and rows of
// the last l blocks), so no two written rows share a ring slot (no races, any thread order). HBM-bound
// copy: 16-byte vectors, one warp per row.
#include "internal.h"

namespace loza {

namespace {

__global__ void __launch_bounds__(256) ring_append_kernel(const uint8_t* __restrict__ rows, int64_t r_sb,
                                                          int64_t r_st, int32_t m, const int32_t* __restrict__ pos0,
                                                          int32_t s, int32_t l, int32_t b, uint8_t* __restrict__ cache,
                                                          int64_t c_sb, int64_t c_st, int32_t batch, int32_t row_bytes) {
  const int64_t total = (int64_t)batch * m;
  const int warps = (int)(blockDim.x >> 5), lane = (int)(threadIdx.x & 31);
  for (int64_t w = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); w < total; w += (int64_t)gridDim.x * warps) {
    const int32_t bi = (int32_t)(w / m), j = (int32_t)(w - (int64_t)bi * m);
    const int64_t p0 = pos0[bi];
    const int64_t pos = p0 + j;
    const int64_t kb = pos / b, last_kb = (p0 + m - 1) / b;
    if (!(kb < s || kb > last_kb - l)) continue;  // evicted before the append completes
    const int64_t dst_row = kb < s ? pos : (int64_t)s * b + ((kb - s) % l) * b + (pos - kb * b);
    const uint4* src = reinterpret_cast<const uint4*>(rows + bi * r_sb + (int64_t)j * r_st);
    uint4* dst = reinterpret_cast<uint4*>(cache + bi * c_sb + dst_row * c_st);
    for (int k = lane; k < row_bytes / 16; k += 32) dst[k] = src[k];
  }
}

}  // namespace

cudaError_t launch_ring_append(const void* rows, int64_t r_sb, int64_t r_st, int32_t m, const int32_t* pos0,
                               int32_t s, int32_t l, int32_t b, void* cache, int64_t c_sb, int64_t c_st,
                               int32_t batch, int32_t row_bytes, cudaStream_t st) {
  const int64_t total = (int64_t)batch * m;
  if (total == 0) return cudaSuccess;
  int64_t blocks = (total + 7) / 8;
  const int64_t cap = (int64_t)device_sm_count() * 8;
  if (blocks > cap) blocks = cap;
  ring_append_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const uint8_t*>(rows), r_sb, r_st, m, pos0,
                                                       s, l, b, reinterpret_cast<uint8_t*>(cache), c_sb, c_st, batch,
                                                       row_bytes);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza
