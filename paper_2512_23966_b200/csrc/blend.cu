// LoZA calibration blend, Eq. 3, and its scalar gradient.
//
//   o_hat = fma(alpha, o_full, (1 - alpha) * o_sparse)    (alpha in {0,1} exact)
//   d_alpha = sum_e d_o_hat[e] * (o_full[e] - o_sparse[e])
//
// HBM-bound elementwise pass: 16-byte vector loads/stores (8 bf16 or 4 fp32),
// grid = 4 x SM count persistent CTAs with a grid-stride loop. The gradient is
// accumulated per thread in fp32, reduced per CTA in fp64 into ws[blockIdx],
// and summed by a second single-CTA kernel in a fixed order (deterministic,
// independent of scheduling). Algorithmic bytes: numel * elem * (2 reads +
// 1 write [+ 1 read of d_o_hat]).
#include "internal.h"

namespace loza {

namespace {

constexpr int kThreads = 512;
constexpr int kMaxBlocks = 148 * 8;

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t rne16(float f) {
  uint32_t u = __float_as_uint(f);
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <bool kBf16, bool kFwd, bool kGrad>
__global__ void __launch_bounds__(kThreads) blend_kernel(const uint4* __restrict__ of, const uint4* __restrict__ os,
                                                         const float* __restrict__ alpha_p, uint4* __restrict__ oh,
                                                         const uint4* __restrict__ dh, double* __restrict__ part,
                                                         int64_t nvec, int32_t* status) {
  const float a = *alpha_p;
  const bool bad = !(a >= 0.f && a <= 1.f);  // NaN fails both
  const float om = 1.f - a;
  float g = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += stride) {
    const uint4 x = ldg_stream(of + i);
    const uint4 y = ldg_stream(os + i);
    uint4 d;
    if (kGrad) d = ldg_stream(dh + i);
    const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
    const uint32_t yw[4] = {y.x, y.y, y.z, y.w};
    uint32_t dw[4] = {0, 0, 0, 0};
    if (kGrad) { dw[0] = d.x; dw[1] = d.y; dw[2] = d.z; dw[3] = d.w; }
    uint32_t rw[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (kBf16) {
        const float x0 = bf_lo(xw[c]), x1 = bf_hi(xw[c]);
        const float y0 = bf_lo(yw[c]), y1 = bf_hi(yw[c]);
        if (kFwd) rw[c] = rne16(fmaf(a, x0, om * y0)) | (rne16(fmaf(a, x1, om * y1)) << 16);
        if (kGrad) g = fmaf(bf_lo(dw[c]), x0 - y0, fmaf(bf_hi(dw[c]), x1 - y1, g));
      } else {
        const float x0 = __uint_as_float(xw[c]), y0 = __uint_as_float(yw[c]);
        if (kFwd) rw[c] = __float_as_uint(fmaf(a, x0, om * y0));
        if (kGrad) g = fmaf(__uint_as_float(dw[c]), x0 - y0, g);
      }
    }
    if (kFwd) oh[i] = make_uint4(rw[0], rw[1], rw[2], rw[3]);
  }
  if (kGrad) {
    double gd = (double)g;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gd += __shfl_xor_sync(0xffffffffu, gd, o);
    __shared__ double wsum[kThreads / 32];
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = gd;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) t += wsum[w];
      part[blockIdx.x] = t;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && status) *status = bad ? LOZA_ERR_INVALID : LOZA_OK;
}

__global__ void dalpha_reduce_kernel(const double* __restrict__ part, int n, const float* __restrict__ alpha_p,
                                     double* __restrict__ out) {
  __shared__ double sh[32];
  double t = 0.0;
  // fixed assignment: lane-strided, then fixed-order tree -> deterministic
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += part[i];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    const float a = *alpha_p;
    *out = (a >= 0.f && a <= 1.f) ? s : __longlong_as_double(0x7FF8000000000000ll);
  }
}

template <bool kBf16>
cudaError_t launch_t(const void* of, const void* os, const float* alpha, void* oh, const void* dh, double* dal,
                     int64_t numel, int32_t* status, void* ws, cudaStream_t st) {
  const int64_t nvec = numel / (kBf16 ? 8 : 4);
  int64_t blocks = (nvec + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)device_sm_count() * 4;
  if (blocks > cap) blocks = cap;
  if (blocks > kMaxBlocks) blocks = kMaxBlocks;
  if (blocks < 1) blocks = 1;
  const bool fwd = oh != nullptr, grad = (dh != nullptr && dal != nullptr);
  double* part = reinterpret_cast<double*>(ws);
  auto a = reinterpret_cast<const uint4*>(of);
  auto b = reinterpret_cast<const uint4*>(os);
  auto c = reinterpret_cast<uint4*>(oh);
  auto d = reinterpret_cast<const uint4*>(dh);
  if (fwd && grad)
    blend_kernel<kBf16, true, true><<<(unsigned)blocks, kThreads, 0, st>>>(a, b, alpha, c, d, part, nvec, status);
  else if (fwd)
    blend_kernel<kBf16, true, false><<<(unsigned)blocks, kThreads, 0, st>>>(a, b, alpha, c, d, part, nvec, status);
  else
    blend_kernel<kBf16, false, true><<<(unsigned)blocks, kThreads, 0, st>>>(a, b, alpha, c, d, part, nvec, status);
  count_launch();
  if (grad) {
    dalpha_reduce_kernel<<<1, 256, 0, st>>>(part, (int)blocks, alpha, dal);
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace

size_t blend_ws_bytes() { return sizeof(double) * kMaxBlocks; }

cudaError_t launch_dalpha_reduce(const double* part, int n, const float* alpha, double* out, cudaStream_t st) {
  dalpha_reduce_kernel<<<1, 256, 0, st>>>(part, n, alpha, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_blend(const void* o_full, const void* o_sparse, const float* alpha, void* o_hat,
                         const void* d_o_hat, double* d_alpha, int64_t numel, int bf16, int32_t* status,
                         void* ws, cudaStream_t st) {
  if (bf16) return launch_t<true>(o_full, o_sparse, alpha, o_hat, d_o_hat, d_alpha, numel, status, ws, st);
  return launch_t<false>(o_full, o_sparse, alpha, o_hat, d_o_hat, d_alpha, numel, status, ws, st);
}

}  // namespace loza
