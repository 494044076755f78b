// UMMA rate per shape with a lean warp-uniform issue loop (no commits inside the loop).
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace loza::sm100;

template <int CG, int M, int N, bool AMN = false, bool BMN = false>
__global__ void __launch_bounds__(128, 1) bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc<CG>(smem_u32(&tptr), 512);
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  constexpr uint32_t idesc = idesc_bf16_f32(M, N, AMN, BMN);
  const bool leader = CG == 1 || cluster_ctarank() == 0;
  if (threadIdx.x < 32 && leader) {
    unsigned long long t0 = clock64();
    const uint64_t a_base = sdesc_sw128(sb, 16, 1024), b_base = sdesc_sw128(sb + 65536, 16, 1024);
    for (int it = 0; it < iters; ++it) {
      const int k = it & 3;
      const uint64_t ad = a_base + (uint64_t)((((it & 7) * 8192 + k * 32)) >> 4);
      const uint64_t bd = b_base + (uint64_t)((((it & 3) * 16384 + k * 32)) >> 4);
      if (elect_one()) {
        if (CG == 2) umma_bf16_pair(tmem, ad, bd, idesc, it > 0);
        else umma_bf16_1sm(tmem, ad, bd, idesc, it > 0);
      }
      __syncwarp();
    }
    if (elect_one()) { if (CG == 2) umma_commit_pair_mc(smem_u32(&bar), 3); else umma_commit_1sm(smem_u32(&bar)); }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  if (CG == 2 && threadIdx.x < 32 && !leader) mbar_wait(smem_u32(&bar), 0);
  __syncwarp();
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<CG>(tmem, 512); }
}

template <int CG, int M, int N, bool AMN = false, bool BMN = false>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(bench<CG, M, N, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  const int iters = 8192;
  cudaLaunchKernelEx(&cfg, bench<CG, M, N, AMN, BMN>, iters, d);
  cudaLaunchKernelEx(&cfg, bench<CG, M, N, AMN, BMN>, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  double sum = 0; int n = 0;
  for (int i = 0; i < 148; i += CG) { sum += h[i]; ++n; }
  const double per = sum / n / iters;
  printf("%-16s err=%d cyc/MMA=%7.1f  MAC/clk/SM=%7.1f (ideal 4096)\n", name, (int)e, per, (double)M * N * 16 / per / CG);
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // the decode kernel's shapes: S^T (K-major A and B) and O^T += V^T P (MN-major A and B)
    run<1, 128, 64>("cg1 M128 N64 KK");
    run<1, 128, 64, true, true>("cg1 M128 N64 MM");
    run<1, 128, 64, false, true>("cg1 M128 N64 KM");
    run<1, 128, 64, true, false>("cg1 M128 N64 MK");
    run<2, 256, 64>("cg2 M256 N64 KK");
    run<2, 256, 64, true, true>("cg2 M256 N64 MM");
    run<1, 128, 128, true, true>("cg1 M128 N128 MM");
    run<2, 128, 256, false, true>("cg2 M128 N256 KM");
    return 0;
  }
  run<1, 64, 64>("cg1 M64 N64");
  run<1, 64, 128>("cg1 M64 N128");
  run<1, 64, 256>("cg1 M64 N256");
  run<1, 128, 64>("cg1 M128 N64");
  run<1, 128, 128>("cg1 M128 N128");
  run<1, 128, 256>("cg1 M128 N256");
  run<2, 128, 128>("cg2 M128 N128");
  run<2, 128, 256>("cg2 M128 N256");
  run<2, 256, 64>("cg2 M256 N64");
  run<2, 256, 128>("cg2 M256 N128");
  run<2, 256, 256>("cg2 M256 N256");
  return 0;
}
