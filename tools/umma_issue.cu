// Issue-path costs of the prefill MMA warp: cta_group::2 M128 N256 K16 UMMAs issued by one warp-uniform
// loop (elected lane), in groups of G UMMAs; per group optionally: wait on an (already completed) mbarrier
// with try_wait or test_wait, tcgen05 fence, one or two commits. Optional interference from 8 warps doing
// TMEM loads (the softmax reading S) or st.shared (P stores). Reports cycles per UMMA (64 = tensor bound).
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace loza::sm100;

enum : int { kWaitTry = 1, kWaitTest = 2, kFence = 4, kCommit2 = 8, kIntTmem = 16, kIntSt = 32, kNoCommit = 64 };

__global__ void __launch_bounds__(352, 1) __cluster_dims__(2, 1, 1)
    bench(int flags, int group, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t done_bar, tbar, ready;
  __shared__ uint32_t tptr;
  __shared__ volatile int stop;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&done_bar), 1);
    mbar_init(smem_u32(&tbar), 1);
    mbar_init(smem_u32(&ready), 1);
    mbar_arrive_local(smem_u32(&ready));  // phase 0 complete: waits with parity 0 return at once
    stop = 0;
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 1) tmem_alloc<2>(smem_u32(&tptr), 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tptr;
  const uint32_t idesc = idesc_bf16_f32(128, 256, false, false);
  const bool leader = cluster_ctarank() == 0;
  if (warp == 1) {
    if (leader) {
      unsigned long long t0 = clock64();
      const uint64_t a_base = sdesc_sw128(sb, 16, 1024), b_base = sdesc_sw128(sb + 73728, 16, 1024);
      for (int it = 0; it < iters; it += group) {
        if (flags & kWaitTry) mbar_wait(smem_u32(&ready), 0);
        if (flags & kWaitTest) while (!mbar_test(smem_u32(&ready), 0)) {}
        if (flags & kFence) tc_fence_after();
        if (elect_one()) {
          for (int g = 0; g < group; ++g) {
            const int k = (it + g) & 3;
            const uint64_t ad = a_base + (uint64_t)(((((it + g) >> 2) % 9) * 8192 + k * 32) >> 4);
            const uint64_t bd = b_base + (uint64_t)(((((it + g) >> 2) % 7) * 16384 + k * 32) >> 4);
            umma_bf16_pair(tmem + 256, ad, bd, idesc, (it + g) > 0);
          }
          if (!(flags & kNoCommit)) umma_commit_pair_mc(smem_u32(&tbar), 3);
          if (flags & kCommit2) umma_commit_pair_mc(smem_u32(&tbar), 3);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit_pair_mc(smem_u32(&done_bar), 3);
      __syncwarp();
      mbar_wait(smem_u32(&done_bar), 0);
      unsigned long long t1 = clock64();
      if (lane == 0) out[blockIdx.x] = t1 - t0;
    } else {
      mbar_wait(smem_u32(&done_bar), 0);
    }
    if (lane == 0) stop = 1;
  } else if (warp >= 2 && warp < 10 && (flags & kIntTmem)) {
    // like the softmax: each warp reads 64 fp32 columns of its lane quarter from the other S buffer (cols 0..255)
    const uint32_t ta = tmem + (((warp & 3) * 32) << 16) + 64 * ((warp - 2) >> 2);
    while (!stop) {
      uint32_t v[32], w[32];
      tmem_ld32(ta, v);
      tmem_ld32(ta + 32, w);
      tmem_wait_ld();
      if (v[0] == 12345u && w[3] == 7u) out[1000] = v[1];
    }
  } else if (warp >= 2 && warp < 10 && (flags & kIntSt)) {
    const uint32_t base = sb + 200 * 1024 - 32768 + (warp - 2) * 4096;
    int i = 0;
    while (!stop) {
      st_shared_v4(base + ((lane * 16 + i * 512) & 4095), i, i, i, i);
      ++i;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 2048 * 8);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct Case {
    const char* name;
    int flags, group;
  } cases[] = {
      {"no commit", kNoCommit, 4},
      {"commit/4", 0, 4},
      {"commit/8", 0, 8},
      {"2 commits/4", kCommit2, 4},
      {"try_wait + commit/4", kWaitTry, 4},
      {"test_wait + commit/4", kWaitTest, 4},
      {"try_wait + fence + commit/4", kWaitTry | kFence, 4},
      {"try_wait + fence + commit/8", kWaitTry | kFence, 8},
      {"try_wait+fence+commit/4 +TMEM ld", kWaitTry | kFence | kIntTmem, 4},
      {"try_wait+fence+commit/4 +st.shared", kWaitTry | kFence | kIntSt, 4},
      {"commit/4 +TMEM ld", kIntTmem, 4},
      {"commit/8 +TMEM ld", kIntTmem, 8},
  };
  for (const Case& c : cases) {
    const int iters = 8192;
    for (int rep = 0; rep < 2; ++rep) bench<<<148, 352, smem>>>(c.flags, c.group, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    int n = 0;
    for (int i = 0; i < 148; i += 2) { s += h[i]; ++n; }
    printf("%-38s err=%d  cyc/UMMA=%6.1f\n", c.name, (int)e, s / n / iters);
  }
  return 0;
}
