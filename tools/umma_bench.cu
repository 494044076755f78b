// Microbenchmark: issue rate of tcgen05.mma for the shapes the kernels use (no TMA, smem preloaded with zeros).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2512_23966_b200/csrc tools/umma_bench.cu -o tools/umma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace loza::sm100;

struct Cfg {
  int cg, M, N, a_mn, b_mn;
  unsigned a_lbo, a_sbo, b_lbo, b_sbo;
  int kstep_bytes_a, kstep_bytes_b;  // descriptor advance per K=16 step
};

template <int CG>
__global__ void __launch_bounds__(128, 1) bench(Cfg c, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc<CG>(smem_u32(&tptr), 512);
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  const uint32_t idesc = idesc_bf16_f32(c.M, c.N, c.a_mn, c.b_mn);
  const bool leader = CG == 1 || cluster_ctarank() == 0;
  if (threadIdx.x < 32 && leader) {  // whole warp runs the loop; one elected lane issues
    unsigned long long t0 = clock64();
    const uint64_t a_base = sdesc_sw128(sb, c.a_lbo, c.a_sbo), b_base = sdesc_sw128(sb + 65536, c.b_lbo, c.b_sbo);
    for (int it = 0; it < iters; ++it) {
      const int k = it & 3;
      const uint64_t ad = a_base + (uint64_t)(((it & 7) * 8192 + k * c.kstep_bytes_a) >> 4);
      const uint64_t bd = b_base + (uint64_t)(((it & 7) * 8192 + k * c.kstep_bytes_b) >> 4);
      if (elect_one()) {
        if (CG == 2) umma_bf16_pair(tmem, ad, bd, idesc, it > 0);
        else umma_bf16_1sm(tmem, ad, bd, idesc, it > 0);
      }
      __syncwarp();
    }
    if (elect_one()) {
      if (CG == 2) umma_commit_pair_mc(smem_u32(&bar), 3);
      else umma_commit_1sm(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  if (CG == 2 && threadIdx.x < 32 && !leader) mbar_wait(smem_u32(&bar), 0);
  __syncwarp();
  tc_fence_before();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem, 512);
  }
}

template <int CG>
void run(const char* name, Cfg c, int grid) {
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  cudaMemset(d, 0, grid * 8);
  const int smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(bench<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int iters = 4096;
  cudaLaunchKernelEx(&cfg, bench<CG>, c, iters, d);
  cudaLaunchKernelEx(&cfg, bench<CG>, c, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[512];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0;
  int n = 0;
  for (int i = 0; i < grid; ++i)
    if (h[i]) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; ++n; }
  const double per = sum / n / iters;
  const double macs = (double)c.M * c.N * 16;  // per instruction (whole pair for cg2)
  printf("%-34s err=%d  cyc/MMA=%7.1f  MAC/clk/SM=%7.1f (ideal 4096)\n", name, (int)e, per, macs / per / CG);
  cudaFree(d);
}

int main() {
  // S: cg2 M128 N128, A/B K-major SW128 (kernel's QK^T)
  run<2>("cg2 M128 N128 KK (S)", Cfg{2, 128, 128, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  run<2>("cg2 M128 N128 KK (S) 1 pair", Cfg{2, 128, 128, 0, 0, 16, 1024, 16, 1024, 32, 32}, 2);
  // PV: cg2 M128 N256, A K-major, B MN-major (LBO 4096, SBO 1024, +2048 per K=16)
  run<2>("cg2 M128 N256 K,MN (PV)", Cfg{2, 128, 256, 0, 1, 16, 1024, 4096, 1024, 32, 2048}, 148);
  run<2>("cg2 M128 N256 KK", Cfg{2, 128, 256, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  run<2>("cg2 M256 N256 KK", Cfg{2, 256, 256, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  run<2>("cg2 M256 N128 KK", Cfg{2, 256, 128, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  run<1>("cg1 M128 N256 KK", Cfg{1, 128, 256, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  run<1>("cg1 M128 N128 KK", Cfg{1, 128, 128, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  run<1>("cg1 M64 N128 KK (decode S)", Cfg{1, 64, 128, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  run<1>("cg1 M64 N256 K,MN (decode PV)", Cfg{1, 64, 256, 0, 1, 16, 1024, 4096, 1024, 32, 2048}, 148);
  run<1>("cg1 M128 N64 KK", Cfg{1, 128, 64, 0, 0, 16, 1024, 16, 1024, 32, 32}, 148);
  return 0;
}
