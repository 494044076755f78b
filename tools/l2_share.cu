// L2 -> SM TMA throughput vs. how many CTAs read the same rows at the same time ("share"), and vs. the
// number of 16 KB loads in flight per SM ("slots"). 148 CTAs, L2-resident 18.9 MB source.
#include <cstdio>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "sm100.cuh"
using namespace loza::sm100;

__global__ void __launch_bounds__(64, 1) bw(const __grid_constant__ CUtensorMap map, int n, int share, int slots,
                                            int loads, int pol_mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb0 = smem_u32(smem);
  const uint32_t sb = (pol_mode & 4) ? ((sb0 + 1023) & ~1023u) : sb0;
  __shared__ uint64_t full[12];
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2000] = sb0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) mbar_init(smem_u32(&full[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pol_mode &= 3;
    const uint64_t pol = pol_mode == 0 ? policy_evict_first() : (pol_mode == 1 ? policy_evict_last() : policy_evict_normal());
    const int base = ((blockIdx.x / share) * 1024) % n;
    unsigned long long t0 = clock64();
    for (int s = 0; s < slots; ++s) {
      mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
      tma_load_3d(sb + s * 16384, &map, (s % 9) * 64, (base + (s / 9) * 128) % n, 0, smem_u32(&full[s]), pol);
    }
    for (int it = 0; it < loads; ++it) {
      const int s = it % slots;
      mbar_wait(smem_u32(&full[s]), (it / slots) & 1);
      const int nx = it + slots;
      if (nx < loads) {
        mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
        tma_load_3d(sb + s * 16384, &map, (nx % 9) * 64, (base + (nx / 9) * 128) % n, 0, smem_u32(&full[s]), pol);
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

template <int S>
__global__ void __launch_bounds__(64, 1) bw_old(const __grid_constant__ CUtensorMap map, int rows_per_cta, int rows_total,
                                            int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t full[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(smem_u32(&full[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    unsigned long long t0 = clock64();
    const int base = (blockIdx.x * rows_per_cta) % rows_total;
    for (int s = 0; s < S; ++s) {
      mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
      tma_load_3d(sb + s * 16384, &map, (s % 9) * 64, (base + (s / 9) * 128) % rows_total, 0, smem_u32(&full[s]), pol);
    }
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(smem_u32(&full[s]), (it / S) & 1);
      const int nx = it + S;
      mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
      tma_load_3d(sb + s * 16384, &map, (nx % 9) * 64, (base + (nx / 9) * 128) % rows_total, 0, smem_u32(&full[s]), pol);
    }
    for (int it = iters; it < iters + S; ++it) mbar_wait(smem_u32(&full[it % S]), (it / S) & 1);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
  }
}

int main() {
  const int n = 16384;
  void* g;
  cudaMalloc(&g, (size_t)n * 1152);
  cudaMemset(g, 0, (size_t)n * 1152);
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
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
  const int smem = 12 * 16384 + 1024;
  cudaFuncSetAttribute(bw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int loads = 2048;
  cudaFuncSetAttribute(bw_old<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rpc : {0, 128, 1024}) {
    for (int rep = 0; rep < 2; ++rep) bw_old<8><<<148, 64, smem>>>(map, rpc, n, loads, d);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    printf("old kernel rows_per_cta=%4d  B/clk/SM=%6.1f\n", rpc, 16384.0 * loads / (cyc / 148));
  }
  const char* pn[] = {"evict_first", "evict_last", "evict_normal"};
  for (int clus : {1, 2})
    for (int pm : {0, 1, 4, 5})
      for (int share : {1, 148}) {
        const int slots = 8;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = clus;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, bw, map, n, share, slots, loads, pm, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, bw, map, n, share, slots, loads, pm, d);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[148];
        cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < 148; ++i) cyc += h[i];
        cyc /= 148;
        unsigned long long sbh; cudaMemcpy(&sbh, d + 2000, 8, cudaMemcpyDeviceToHost);
        printf("sb0&1023=%4llu aligned=%d ", sbh & 1023, pm >> 2);
        printf("cluster=%d %-12s share=%3d err=%d  B/clk/SM=%6.1f  aggregate=%7.1f GB/s\n", clus, pn[pm & 3], share, (int)err,
               16384.0 * loads / cyc, 16384.0 * loads * 148 / (ms * 1e-3) / 1e9);
      }
  return 0;
}
