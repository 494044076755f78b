// Shared-memory bandwidth sharing between the tensor pipe and TMA: cta_group::2 M128 N256 K16 UMMAs
// (operands in smem, 96 B/clk/SM of operand reads at full rate) run back to back while a TMA ring
// (4 x 16 KB, L2-resident source) streams into another smem region. Reports the UMMA rate and the TMA
// fill rate, alone and together.
#include <cstdio>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "sm100.cuh"

using namespace loza::sm100;

__global__ void __launch_bounds__(128, 1) __cluster_dims__(2, 1, 1)
    bench(int mode, int iters, unsigned long long* out, const __grid_constant__ CUtensorMap map, int n) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t bar, tbar, full[4];
  __shared__ uint32_t tptr;
  __shared__ volatile int stop;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&tbar), 1);
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&full[i]), 1);
    stop = 0;
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<2>(smem_u32(&tptr), 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tptr;
  const uint32_t idesc = idesc_bf16_f32(128, 256, false, false);
  const bool leader = cluster_ctarank() == 0;
  const bool do_mma = mode != 1, do_tma = mode != 0;
  if (warp == 0) {
    if (do_mma) {
      if (leader) {
        unsigned long long t0 = clock64();
        const uint64_t a_base = sdesc_sw128(sb, 16, 1024), b_base = sdesc_sw128(sb + 65536, 16, 1024);
        for (int it = 0; it < iters; ++it) {
          const int k = it & 3;
          const uint64_t ad = a_base + (uint64_t)((((it & 7) * 8192 + k * 32)) >> 4);
          const uint64_t bd = b_base + (uint64_t)((((it & 3) * 16384 + k * 32)) >> 4);
          if (elect_one()) umma_bf16_pair(tmem, ad, bd, idesc, it > 0);
          __syncwarp();
          if ((it & 3) == 3) {
            if (elect_one()) umma_commit_pair_mc(smem_u32(&tbar), 3);
            __syncwarp();
          }
        }
        if (elect_one()) umma_commit_pair_mc(smem_u32(&bar), 3);
        __syncwarp();
        mbar_wait(smem_u32(&bar), 0);
        unsigned long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = t1 - t0;
      } else {
        mbar_wait(smem_u32(&bar), 0);
      }
      if (lane == 0) stop = 1;
    }
  } else if (warp == 1 && do_tma) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      const uint32_t ring = sb + 131072;
      int row = (blockIdx.x * 1024) & (n - 1), cc = 0;
      unsigned long long t0 = clock64();
      for (int s = 0; s < 4; ++s) {
        mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
        tma_load_3d(ring + s * 16384, &map, cc * 64, row, 0, smem_u32(&full[s]), pol);
        if (++cc == 9) { cc = 0; row = (row + 128) & (n - 1); }
      }
      const int max_loads = 6000;  // ~ the UMMA run length at ~100 B/clk
      int loads = 0;
      for (int it = 0;; ++it) {
        const int s = it & 3;
        mbar_wait(smem_u32(&full[s]), (it >> 2) & 1);
        ++loads;
        if (loads >= max_loads) break;
        mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
        tma_load_3d(ring + s * 16384, &map, cc * 64, row, 0, smem_u32(&full[s]), pol);
        if (++cc == 9) { cc = 0; row = (row + 128) & (n - 1); }
      }
      for (int it = loads; it < loads + 3; ++it) mbar_wait(smem_u32(&full[it & 3]), (it >> 2) & 1);
      loads += 3;
      unsigned long long t1 = clock64();
      out[512 + blockIdx.x] = t1 - t0;
      out[1024 + blockIdx.x] = loads;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 2048 * 8);
  cudaMemset(d, 0, 2048 * 8);
  const int n = 16384;
  void* g;
  cudaMalloc(&g, (size_t)n * 576 * 2);
  cudaMemset(g, 0, (size_t)n * 576 * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[3] = {576, (cuuint64_t)n, 1};
  cuuint64_t strides[2] = {1152, (cuuint64_t)1152 * n};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"UMMA only", "TMA only", "UMMA + TMA"};
  for (int mode = 0; mode < 3; ++mode) {
    const int iters = 16384;
    for (int rep = 0; rep < 2; ++rep) bench<<<148, 128, smem>>>(mode, iters, d, map, n);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2048];
    cudaMemcpy(h, d, 2048 * 8, cudaMemcpyDeviceToHost);
    double mc = 0, tc = 0, tl = 0;
    int nm = 0, nt = 0;
    for (int i = 0; i < 148; ++i) {
      if (mode != 1 && (i & 1) == 0) { mc += h[i]; ++nm; }
      if (mode != 0) { tc += h[512 + i]; tl += h[1024 + i]; ++nt; }
    }
    printf("%-12s err=%d", names[mode], (int)e);
    if (nm) printf("  UMMA cyc/instr=%6.1f (ideal 64)  smem operand B/clk=%6.1f", mc / nm / iters, 6144.0 / (mc / nm / iters));
    if (nt) printf("  TMA B/clk/SM=%6.1f", tl * 16384.0 / tc);
    printf("\n");
  }
  return 0;
}
