// Per-launch floor inside a CUDA graph for the decode grid shape: 128 CTAs, cluster 2, ~227 KB dynamic smem,
// 320 threads, TMEM alloc/dealloc, vs a plain small kernel.
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace loza::sm100;
__global__ void __launch_bounds__(320, 1) __cluster_dims__(2, 1, 1) k_cluster(int* out, int tmem_on) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tp;
  if (tmem_on && threadIdx.x < 32) tmem_alloc<1>(smem_u32(&tp), 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = smem[0];
  __syncthreads();
  if (tmem_on && threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<1>(tp, 512); }
}
__global__ void k_plain(int* out) { if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = 1; }
int main() {
  int* d; cudaMalloc(&d, 4);
  const int smem = 221 * 1024;  // + static smem stays under the 227 KB limit
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  k_cluster<<<128, 320, smem, s>>>(d, 1); printf("eager launch: %s\n", cudaGetErrorString(cudaStreamSynchronize(s)));
  for (int mode = 0; mode < 3; ++mode) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaGetLastError();
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 64; ++i) {
      if (mode == 0) k_plain<<<128, 320, 0, s>>>(d);
      else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(128); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = smem; cfg.stream = s;
        cudaLaunchKernelEx(&cfg, k_cluster, d, (int)(mode == 2));
      }
    }
    cudaError_t ce = cudaStreamEndCapture(s, &g);
    if (ce != cudaSuccess) { printf("capture failed: %s\n", cudaGetErrorString(ce)); cudaGetLastError(); continue; }
    ce = cudaGraphInstantiate(&ge, g, 0);
    if (ce != cudaSuccess) { printf("instantiate failed: %s\n", cudaGetErrorString(ce)); cudaGetLastError(); continue; }
    for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %.2f us per launch (err %d)\n", mode == 0 ? "plain 128x320" : (mode == 1 ? "cluster2 227KB" : "cluster2 227KB + TMEM alloc"),
           ms * 1e3 / 640, (int)cudaGetLastError());
  }
  return 0;
}
