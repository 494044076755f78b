// Which TMEM (lane, column, half) does a cta_group::2 M128 UMMA read for A[m][k] when A comes from TMEM?
// (The MLA prefill's UMMAs are M128 cg2: 64 rows per CTA, D folded as lanes 0-63 = N half 0, 64-127 = N half 1.)
// B = identity (K-major SW128, N = 32: each CTA provides 16 rows), so D[m][n] = A[m][n mod 16]. Run 0 fills
// TMEM A with value = lane + 1, run 1 with value = 2 * column + half + 1 (bf16-exact); D reveals the mapping.
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace loza::sm100;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ uint16_t bf(float x) { return (uint16_t)(__float_as_uint(x) >> 16); }

__global__ void __launch_bounds__(128, 1) __cluster_dims__(2, 1, 1) probe(int run, float* out) {
  __shared__ __align__(1024) uint8_t bsm[16 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, rank = cluster_ctarank();
  // B rows n (16 per CTA), K-major, 64 bf16 per row, SWIZZLE_128B: B[n][k] = (n == k)
  for (int i = threadIdx.x; i < 16 * 64; i += 128) {
    const int n = i / 64, k = i % 64;
    const uint32_t off = n * 128 + ((((k * 2) >> 4) ^ (n & 7)) << 4) + (k * 2) % 16;
    *reinterpret_cast<uint16_t*>(bsm + off) = n == k ? bf(1.0f) : 0;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<2>(smem_u32(&tptr), 128);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tptr;
  // A region: columns [0, 8) of every lane
  {
    uint32_t v[8];
    const uint32_t ln = 32 * warp + lane;
    for (int c = 0; c < 8; ++c) {
      const float lo = run == 0 ? (float)(ln + 1) : (float)(2 * c + 1);
      const float hi = run == 0 ? (float)(ln + 1) : (float)(2 * c + 2);
      v[c] = (uint32_t)bf(lo) | ((uint32_t)bf(hi) << 16);
    }
    tmem_st8(tmem + ((32 * warp) << 16), v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (rank == 0 && warp == 0) {
    const uint64_t bd = sdesc_sw128(smem_u32(bsm), 16, 1024);
    constexpr uint32_t idesc = idesc_bf16_f32(128, 32, false, false);
    if (elect_one()) {
      umma_bf16_pair_ts(tmem + 64, tmem, bd, idesc, 0);
      umma_commit_pair_mc(smem_u32(&bar), 3);
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  uint32_t d[32];
  tmem_ld32(tmem + ((32 * warp) << 16) + 64, d);
  tmem_wait_ld();
  const uint32_t ln = 32 * warp + lane;
  for (int j = 0; j < 32; ++j) out[(rank * 128 + ln) * 32 + j] = __uint_as_float(d[j]);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 128);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 2 * 128 * 32 * 4);
  static float h[2][2 * 128 * 32];
  for (int run = 0; run < 2; ++run) {
    cudaMemset(d, 0, 2 * 128 * 32 * 4);
    probe<<<2, 128>>>(run, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("run %d: %s\n", run, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h[run], d, sizeof(h[run]), cudaMemcpyDeviceToHost);
  }
  // D lane L, column j (of the 32 read): print (A lane, A column/half) per (CTA, D lane, D column)
  for (int cta = 0; cta < 2; ++cta)
    for (int L = 0; L < 128; L += (L < 4 || (L >= 60 && L < 68) || L > 124) ? 1 : 8) {
      printf("cta %d Dlane %3d:", cta, L);
      for (int j = 0; j < 18; ++j) {
        const float a = h[0][(cta * 128 + L) * 32 + j], b = h[1][(cta * 128 + L) * 32 + j];
        printf(" %3.0f/%2.0f", a, b);
      }
      printf("\n");
    }
  return 0;
}
