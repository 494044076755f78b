// TMA receive bandwidth per SM: a ring of S stages x 16 KB (box {64, 128} bf16, SW128), one producer thread,
// the consumer simply releases each stage when it lands. Data: a [rows, 576] bf16 tensor; each CTA walks
// its own rows (HBM-resident: 1.2 GB tensor, or L2-resident: 16 MB tensor).
#include <cstdio>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "sm100.cuh"
using namespace loza::sm100;

template <int S>
__global__ void __launch_bounds__(64, 1) bw(const __grid_constant__ CUtensorMap map, int rows_per_cta, int rows_total,
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
    long long bytes = 0;
    const int base = (blockIdx.x * rows_per_cta) % rows_total;
    // prime
    for (int s = 0; s < S; ++s) {
      mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
      tma_load_3d(sb + s * 16384, &map, (s % 9) * 64, (base + (s / 9) * 128) % rows_total, 0, smem_u32(&full[s]), pol);
    }
    for (int it = 0; it < iters; ++it) {
      const int s = it % S;
      mbar_wait(smem_u32(&full[s]), (it / S) & 1);
      bytes += 16384;
      const int nx = it + S;
      mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
      tma_load_3d(sb + s * 16384, &map, (nx % 9) * 64, (base + (nx / 9) * 128) % rows_total, 0, smem_u32(&full[s]), pol);
    }
    for (int it = iters; it < iters + S; ++it) mbar_wait(smem_u32(&full[it % S]), (it / S) & 1);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = (t1 - t0);
    out[1024 + blockIdx.x] = bytes;
  }
}

int main() {
  void* g;
  const long long rows = 1 << 20;  // 1M rows x 1152 B = 1.2 GB
  cudaMalloc(&g, rows * 1152);
  cudaMemset(g, 0, rows * 1152);
  unsigned long long* d;
  cudaMalloc(&d, 4096 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  for (int l2 = 0; l2 < 2; ++l2) {
    const long long r = l2 ? 16384 : rows;  // L2-resident (18.9 MB) or HBM-resident
    CUtensorMap map;
    cuuint64_t dims[3] = {576, (cuuint64_t)r, 1};
    cuuint64_t strides[2] = {1152, (cuuint64_t)(1152 * r)};
    cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {1, 64, 128, 148}) {
      for (int S : {4, 8, 12}) {
        const int smem = 13 * 16384;
        const int iters = 2048;
        auto k = S == 4 ? bw<4> : (S == 8 ? bw<8> : bw<12>);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k<<<grid, 64, smem>>>(map, (int)(r / grid / 128) * 128, (int)r, iters, d);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<grid, 64, smem>>>(map, (int)(r / grid / 128) * 128, (int)r, iters, d);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[148];
        cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        double cyc = 0; for (int i = 0; i < grid; ++i) cyc += h[i]; cyc /= grid;
        const double bytes = 16384.0 * iters;
        printf("%s grid=%3d stages=%2d err=%d  B/clk/SM=%6.1f  aggregate=%7.1f GB/s\n", l2 ? "L2 " : "HBM", grid, S,
               (int)err, bytes / cyc, bytes * grid / (ms * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
