// Integer prologue: per query block, the selected key blocks.
// sel(QB) = {kb in [0, QB] : kb < s  or  QB - kb < l}, ascending — the closed form
// of the token mask of Eq. 4 / SPEC.md:121 (a key block holds an allowed key for
// some query of QB iff it is a sink block or one of the l local blocks ending at
// QB; the query's own block is local, "summing to 1,024 tokens").
#include "internal.h"

namespace loza {

__global__ void select_blocks_kernel(int64_t n_qb, int64_t qb0, int32_t s, int32_t l, int32_t* idx,
                                     int32_t* cnt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_qb) return;
  const int64_t QB = qb0 + t;
  const int32_t w = s + l;
  int32_t c = 0;
  // sinks: kb < min(s, QB+1)
  const int64_t sink_end = QB + 1 < s ? QB + 1 : s;
  for (int64_t kb = 0; kb < sink_end; ++kb) idx[t * w + c++] = (int32_t)kb;
  // locals: kb in [max(s, QB-l+1), QB]
  int64_t lo = QB - l + 1;
  if (lo < s) lo = s;
  for (int64_t kb = lo; kb <= QB; ++kb) idx[t * w + c++] = (int32_t)kb;
  cnt[t] = c;
  for (int32_t r = c; r < w; ++r) idx[t * w + r] = -1;
}

cudaError_t launch_select_blocks(int64_t n_q, int64_t q_start, int32_t s, int32_t l, int32_t b,
                                 int32_t* idx, int32_t* cnt, cudaStream_t st) {
  const int64_t n_qb = (n_q + b - 1) / b;
  if (n_qb == 0) return cudaSuccess;
  const int threads = 128;
  select_blocks_kernel<<<(unsigned)((n_qb + threads - 1) / threads), threads, 0, st>>>(n_qb, q_start / b, s, l,
                                                                                        idx, cnt);
  count_launch();
  return cudaGetLastError();
}

}  // namespace loza
