// Microbenchmark: cta_group::2 M128 N256 UMMA rate under interference from concurrent
// (B) TMEM loads, (C) shared-memory stores, (D) TMA loads, (E) random operand data.
#include <cstdio>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "sm100.cuh"

using namespace loza::sm100;

__global__ void __launch_bounds__(256, 1) __cluster_dims__(2, 1, 1)
    bench(int mode, int iters, unsigned long long* out, const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t bar, tbar, bar2;
  __shared__ uint32_t tptr;
  __shared__ volatile int stop;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = (mode == 4) ? (i * 2654435761u) & 0x3F7F3F7Fu : 0u;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_init(smem_u32(&tbar), 1);
    mbar_init(smem_u32(&bar2), 1);
    mbar_arrive_local(smem_u32(&bar2));
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
  if (warp == 0 && mode >= 10) {
    // whole warp runs the loop (uniform registers); one elected lane issues
    if (leader) {
      unsigned long long t0 = clock64();
      const int cevery = mode == 11 ? 4 : (mode == 12 ? 2 : 1 << 30);
      const uint64_t a_base = sdesc_sw128(sb, 16, 1024), b_base = sdesc_sw128(sb + 65536, 16, 1024);
      for (int it = 0; it < iters; ++it) {
        const int k = it & 3;
        const uint64_t ad = a_base + (uint64_t)((((it & 7) * 8192 + k * 32)) >> 4);
        const uint64_t bd = b_base + (uint64_t)((((it & 3) * 16384 + k * 32)) >> 4);
        if (elect_one()) umma_bf16_pair(tmem, ad, bd, idesc, it > 0);
        __syncwarp();
        if ((it & (cevery - 1)) == cevery - 1) {
          if (elect_one()) umma_commit_pair_mc(smem_u32(&tbar), 3);
          __syncwarp();
        }
      }
      if (elect_one()) umma_commit_pair_mc(smem_u32(&bar), 3);
      __syncwarp();
      mbar_wait(smem_u32(&bar), 0);
      unsigned long long t1 = clock64();
      if (lane == 0) out[blockIdx.x] = t1 - t0;
    }
    if (!leader) mbar_wait(smem_u32(&bar), 0);
    __syncwarp();
    if (lane == 0) stop = 1;
  } else if (warp == 0) {
    if (lane == 0 && leader) {
      unsigned long long t0 = clock64();
      const int cevery = mode == 9 ? 4 : (mode >= 5 ? (1 << (mode - 5)) : 1 << 30);  // commit every cevery MMAs
      for (int it = 0; it < iters; ++it) {
        const int k = it & 3;
        const uint64_t ad = sdesc_sw128(sb + (it & 7) * 8192 + k * 32, 16, 1024);
        const uint64_t bd = sdesc_sw128(sb + 65536 + (it & 3) * 16384 + k * 32, 16, 1024);
        umma_bf16_pair(tmem, ad, bd, idesc, it > 0);
        if ((it + 1) % cevery == 0) {
          umma_commit_pair_mc(smem_u32(&tbar), 3);
          if (mode == 9) { mbar_wait(smem_u32(&bar2), 0); tc_fence_after(); }
        }
      }
      umma_commit_pair_mc(smem_u32(&bar), 3);
      mbar_wait(smem_u32(&bar), 0);
      unsigned long long t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    }
    if (lane == 0 && !leader) mbar_wait(smem_u32(&bar), 0);
    __syncwarp();
    if (lane == 0) stop = 1;
  } else if (warp >= 4 && mode == 1) {
    // TMEM loads from the S region (cols 256..511) of this warp's lane quarter
    const uint32_t ta = tmem + (((warp & 3) * 32) << 16) + 256;
    while (!stop) {
      uint32_t v[32];
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        tmem_ld32(ta + 32 * c, v);
        tmem_wait_ld();
      }
      if (v[0] == 12345u) out[1000] = v[1];
    }
  } else if (warp >= 4 && mode == 2) {
    const uint32_t base = sb + 131072 + (warp - 4) * 8192;
    int i = 0;
    while (!stop) {
      st_shared_v4(base + ((lane * 16 + i * 512) & 8191), i, i, i, i);
      ++i;
    }
  } else if (warp == 1 && mode == 3) {
    if (lane == 0) {
      uint32_t ph = 0;
      int row = 0;
      while (!stop) {
        mbar_arrive_expect_tx(smem_u32(&tbar), 16384);
        tma_load_3d(sb + 131072, &map, 0, row, 0, smem_u32(&tbar), policy_evict_last());
        mbar_wait(smem_u32(&tbar), ph);
        ph ^= 1;
        row = (row + 128) & 4095;
      }
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
  void* g;
  cudaMalloc(&g, 4096 * 576 * 2);
  cudaMemset(g, 0, 4096 * 576 * 2);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[3] = {576, 4096, 1};
  cuuint64_t strides[2] = {1152, 1152 * 4096};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = 200 * 1024 + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"baseline", "+TMEM loads (4 warps)", "+st.shared (4 warps)", "+TMA loads", "random data", "commit every 1", "commit every 2", "commit every 4", "commit every 8", "commit4+wait+fence", "warp-uniform, no commit", "warp-uniform, commit/4", "warp-uniform, commit/2"};
  for (int mode = 0; mode < 13; ++mode) {
    const int iters = 8192;
    bench<<<148, 256, smem>>>(mode, iters, d, map);
    bench<<<148, 256, smem>>>(mode, iters, d, map);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double sum = 0;
    int n = 0;
    for (int i = 0; i < 148; i += 2) { sum += h[i]; ++n; }
    const double per = sum / n / iters;
    printf("%-26s err=%d cyc/MMA=%7.1f  MAC/clk/SM=%7.1f\n", names[mode], (int)e, per, 128.0 * 256 * 16 / per / 2);
  }
  return 0;
}
