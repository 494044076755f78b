// TMA fill rate per SM vs. bytes per TMA instruction. A 4-D view {64 dims, rows, 9 chunks, 1} of a
// [rows, 576] bf16 tensor lets one instruction fetch C consecutive 16 KB chunks (box {64, 128, C, 1}).
// Lean issue loop (power-of-two ring, no divisions). 148 CTAs, distinct rows per CTA, L2-resident.
#include <cstdio>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "sm100.cuh"
using namespace loza::sm100;


template <int C, int SLOTS>  // C chunks per instruction; SLOTS instructions in flight
__global__ void __launch_bounds__(64, 1) bw(const __grid_constant__ CUtensorMap map, int n, int loads,
                                            unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t full[SLOTS];
  if (threadIdx.x == 0) {
    for (int i = 0; i < SLOTS; ++i) mbar_init(smem_u32(&full[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_last();
    constexpr int kPerRow = 9 / C;  // instructions per 128-row block (C divides 9 or C == 8 -> 1)
    int row = (blockIdx.x * 1024) & (n - 1), cc = 0;
    unsigned long long t0 = clock64();
    for (int s = 0; s < SLOTS; ++s) {
      mbar_arrive_expect_tx(smem_u32(&full[s]), C * 16384);
      tma_load_4d(sb + s * C * 16384, &map, 0, row, cc * C, 0, smem_u32(&full[s]), pol);
      if (++cc == kPerRow) { cc = 0; row = (row + 128) & (n - 1); }
    }
    for (int it = 0; it < loads; ++it) {
      const int s = it & (SLOTS - 1);
      mbar_wait(smem_u32(&full[s]), (it / SLOTS) & 1);
      mbar_arrive_expect_tx(smem_u32(&full[s]), C * 16384);
      tma_load_4d(sb + s * C * 16384, &map, 0, row, cc * C, 0, smem_u32(&full[s]), pol);
      if (++cc == kPerRow) { cc = 0; row = (row + 128) & (n - 1); }
    }
    for (int it = loads; it < loads + SLOTS; ++it) mbar_wait(smem_u32(&full[it & (SLOTS - 1)]), (it / SLOTS) & 1);
    out[blockIdx.x] = clock64() - t0;
    out[512 + blockIdx.x] = (unsigned long long)(loads + SLOTS) * C * 16384;
  }
}

template <int SLOTS>
__global__ void __launch_bounds__(64, 1) bw3(const __grid_constant__ CUtensorMap map, int n, int loads,
                                             unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t full[SLOTS];
  if (threadIdx.x == 0) {
    for (int i = 0; i < SLOTS; ++i) mbar_init(smem_u32(&full[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_last();
    int row = (blockIdx.x * 1024) & (n - 1), cc = 0;
    unsigned long long t0 = clock64();
    for (int s = 0; s < SLOTS; ++s) {
      mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
      tma_load_3d(sb + s * 16384, &map, cc * 64, row, 0, smem_u32(&full[s]), pol);
      if (++cc == 9) { cc = 0; row = (row + 128) & (n - 1); }
    }
    for (int it = 0; it < loads; ++it) {
      const int s = it & (SLOTS - 1);
      mbar_wait(smem_u32(&full[s]), (it / SLOTS) & 1);
      mbar_arrive_expect_tx(smem_u32(&full[s]), 16384);
      tma_load_3d(sb + s * 16384, &map, cc * 64, row, 0, smem_u32(&full[s]), pol);
      if (++cc == 9) { cc = 0; row = (row + 128) & (n - 1); }
    }
    for (int it = loads; it < loads + SLOTS; ++it) mbar_wait(smem_u32(&full[it & (SLOTS - 1)]), (it / SLOTS) & 1);
    out[blockIdx.x] = clock64() - t0;
    out[512 + blockIdx.x] = (unsigned long long)(loads + SLOTS) * 16384;
  }
}

template <int C, int SLOTS>
void run(const CUtensorMap& map, int n, unsigned long long* d, int grid) {
  const int smem = C * SLOTS * 16384;
  cudaFuncSetAttribute(bw<C, SLOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int loads = 4096 / C;
  for (int rep = 0; rep < 2; ++rep) bw<C, SLOTS><<<grid, 64, smem>>>(map, n, loads, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, d, 1024 * 8, cudaMemcpyDeviceToHost);
  double cyc = 0, by = 0;
  for (int i = 0; i < grid; ++i) { cyc += h[i]; by += h[512 + i]; }
  printf("grid=%3d box=%d chunks (%3d KB) in flight=%2d instr (%3d KB) err=%d  B/clk/SM=%6.1f\n", grid, C, 16 * C,
         SLOTS, 16 * C * SLOTS, (int)e, by / cyc);
}

int main() {
  const int n = 16384;
  void* g;
  cudaMalloc(&g, (size_t)n * 1152);
  cudaMemset(g, 0, (size_t)n * 1152);
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  {
    CUtensorMap m3;
    cuuint64_t d3[3] = {576, (cuuint64_t)n, 1};
    cuuint64_t s3[2] = {1152, (cuuint64_t)1152 * n};
    cuuint32_t b3[3] = {64, 128, 1}, e3[3] = {1, 1, 1};
    ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, d3, s3, b3, e3,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {1, 148})
      for (int cl : {1, 2})
      for (int smem : {4 * 16384, 128 * 1024, 200 * 1024, 227 * 1024}) {
        cudaFuncSetAttribute(bw3<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = grid == 1 ? 1 : cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, bw3<4>, m3, n, 4096, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[1024];
        cudaMemcpy(h, d, 1024 * 8, cudaMemcpyDeviceToHost);
        double cyc = 0, by = 0;
        for (int i = 0; i < grid; ++i) { cyc += h[i]; by += h[512 + i]; }
        printf("3D map grid=%3d cluster=%d smem=%3d KB 4 x 16 KB err=%d  B/clk/SM=%6.1f\n", grid, cl, smem / 1024, (int)e, by / cyc);
      }
  }
  CUtensorMap map;
  cuuint64_t dims[4] = {64, (cuuint64_t)n, 9, 1};
  cuuint64_t strides[3] = {1152, 128, (cuuint64_t)1152 * n};
  for (int C : {1, 2, 4, 8}) {
    cuuint32_t box[4] = {64, 128, (cuuint32_t)C, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, g, dims, strides,
                                                         box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode C=%d failed %d\n", C, (int)r); continue; }
    for (int grid : {1, 148}) {
      if (C == 1) { run<1, 4>(map, n, d, grid); run<1, 8>(map, n, d, grid); }
      if (C == 2) { run<2, 2>(map, n, d, grid); run<2, 4>(map, n, d, grid); }
      if (C == 4) { run<4, 1>(map, n, d, grid); run<4, 2>(map, n, d, grid); }
      if (C == 8) { run<8, 1>(map, n, d, grid); }
    }
  }
  return 0;
}
