// Legacy warp-level MMA (mma.sync m16n8k16 bf16 -> fp32, SASS HMMA) throughput on sm_100a: W warps per CTA,
// C independent accumulator chains per warp, one CTA per SM. Prints MAC/clk/SM and TFLOP/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/hmma_rate tools/hmma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void hmma_loop(float* out, int iters, long long* cyc) {
  float d[C][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u}, b0 = threadIdx.x * 11u,
           b1 = threadIdx.x * 13u;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps, int sms) {
  const int iters = 4096;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * warps * 32);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  hmma_loop<C><<<sms, warps * 32>>>(out, 16, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  hmma_loop<C><<<sms, warps * 32>>>(out, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c0;
  cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
  const double macs_cta = (double)warps * C * iters * 16 * 8 * 16;
  printf("warps %2d chains %d: %7.1f MAC/clk/SM  %7.1f TFLOP/s (all SMs)\n", warps, C, macs_cta / (double)c0,
         2.0 * macs_cta * sms / (ms * 1e-3) / 1e12);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run<1>(w, sms);
    run<2>(w, sms);
    run<4>(w, sms);
    run<8>(w, sms);
  }
  return 0;
}
