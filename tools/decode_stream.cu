// Streaming ceiling of the decode access pattern: 2 CTAs per sequence (B = 64, 128 CTAs), each TMA-loads the cache
// rows its pair-cooperative decode CTA reads (4 pair tiles x one 128-key sub-block x 576 dims = 4 x 147 KB, and
// optionally the V reload of the same tile: 4 x 32 KB from L2) through a ring of S x 32 KB that the consumer
// releases as soon as an item lands. Timed like tools/decode_time.py: a CUDA graph of 64 launches over 4 rotating
// windows, 512 MB L2 flush before each replay. No compute: the bound the decode's memory pipeline could reach.
#include <cstdio>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "sm100.cuh"
using namespace loza::sm100;

constexpr int B = 64, CTX = 131072;

template <int S, bool V>
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap map, int ctx) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t full[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(smem_u32(&full[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int bi = blockIdx.x >> 1, r = blockIdx.x & 1;
  const int pos = ctx - 1, QB = pos / 128;
  auto sub_row = [&](int j) { return j == 0 ? 0 : (QB - 7 + j) * 128; };  // (1,7,128): sink + 7 local blocks
  // item list: per pair tile i: K = 5 items (chunk pairs; the 5th one chunk), then (V) 4 items of 2 x 16 KB
  const uint64_t pol = policy_evict_last();
  int n = 0;
  auto issue = [&](int item, int s) {
    // decode item -> (row, chunk0, nchunks)
    int per = V ? 9 : 5;
    int i = item / per, k = item % per;
    int row, c0, nc;
    if (k < 5) {
      row = sub_row(2 * i + r);
      c0 = 2 * k;
      nc = k < 4 ? 2 : 1;
    } else {
      const int q = k - 5;
      row = sub_row(2 * i + (q >> 1)) + 64 * (q & 1);
      c0 = 4 * r;
      nc = 2;
    }
    mbar_arrive_expect_tx(smem_u32(&full[s]), nc * 16384);
    for (int c = 0; c < nc; ++c)
      tma_load_3d(sb + s * 32768 + c * 16384, &map, 64 * (c0 + c), row, bi, smem_u32(&full[s]), pol);
  };
  const int total = 4 * (V ? 9 : 5);
  for (int s = 0; s < S && s < total; ++s) issue(s, s);
  for (int it = 0; it < total; ++it) {
    const int s = it % S;
    mbar_wait(smem_u32(&full[s]), (it / S) & 1);
    if (it + S < total) issue(it + S, s);
  }
  (void)n;
}


// two rings: K items (HBM) and V items (L2 re-reads) in separate slots with their own producer threads; one
// consumer takes them in the decode's MMA order K(0), K(1), V(0), K(2), V(1), ..., V(3)
template <int SK, int SV>
__global__ void __launch_bounds__(96, 1) stream2(const __grid_constant__ CUtensorMap map, int ctx) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t fullk[SK], emptyk[SK], fullv[SV], emptyv[SV];
  if (threadIdx.x == 0) {
    for (int i = 0; i < SK; ++i) { mbar_init(smem_u32(&fullk[i]), 1); mbar_init(smem_u32(&emptyk[i]), 1); }
    for (int i = 0; i < SV; ++i) { mbar_init(smem_u32(&fullv[i]), 1); mbar_init(smem_u32(&emptyv[i]), 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const int bi = blockIdx.x >> 1, r = blockIdx.x & 1;
  const int pos = ctx - 1, QB = pos / 128;
  auto sub_row = [&](int j) { return j == 0 ? 0 : (QB - 7 + j) * 128; };
  const uint64_t pol = policy_evict_last();
  if (threadIdx.x == 0) {  // K producer: 4 tiles x 5 items
    for (int it = 0; it < 20; ++it) {
      const int s = it % SK;
      if (it >= SK) mbar_wait(smem_u32(&emptyk[s]), ((it / SK) - 1) & 1);
      const int i = it / 5, k = it % 5, nc = k < 4 ? 2 : 1;
      mbar_arrive_expect_tx(smem_u32(&fullk[s]), nc * 16384);
      for (int c = 0; c < nc; ++c)
        tma_load_3d(sb + s * 32768 + c * 16384, &map, 64 * (2 * k + c), sub_row(2 * i + r), bi, smem_u32(&fullk[s]), pol);
    }
  } else if (threadIdx.x == 32) {  // V producer: 4 tiles x 4 items
    for (int it = 0; it < 16; ++it) {
      const int s = it % SV;
      if (it >= SV) mbar_wait(smem_u32(&emptyv[s]), ((it / SV) - 1) & 1);
      const int i = it / 4, q = it % 4;
      mbar_arrive_expect_tx(smem_u32(&fullv[s]), 2 * 16384);
      for (int c = 0; c < 2; ++c)
        tma_load_3d(sb + (SK + s) * 32768 + c * 16384, &map, 64 * (4 * r + c), sub_row(2 * i + (q >> 1)) + 64 * (q & 1),
                    bi, smem_u32(&fullv[s]), pol);
    }
  } else if (threadIdx.x == 64) {  // consumer in MMA order
    int ik = 0, iv = 0;
    auto takek = [&](int n) { for (int j = 0; j < n; ++j, ++ik) { const int s = ik % SK; mbar_wait(smem_u32(&fullk[s]), (ik / SK) & 1); mbar_arrive_local(smem_u32(&emptyk[s])); } };
    auto takev = [&](int n) { for (int j = 0; j < n; ++j, ++iv) { const int s = iv % SV; mbar_wait(smem_u32(&fullv[s]), (iv / SV) & 1); mbar_arrive_local(smem_u32(&emptyv[s])); } };
    takek(5);
    for (int i = 1; i < 4; ++i) { takek(5); takev(4); }
    takev(4);
  }
}

// one ring, items in the interleaved order K(0), K(1), V(0)a, K(2)a, V(0)b, K(2)b, V(1)a, K(3)a, V(1)b, K(3)b, V(2),
// V(3) (a = first 2 items, b = the rest): the MMA would issue half of PV(i), the first K items of S(i + 2), then
// the rest, so K(i + 2) is in flight while P(i) is being made
template <int S>
__global__ void __launch_bounds__(64, 1) stream3(const __grid_constant__ CUtensorMap map, int ctx) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  __shared__ uint64_t full[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(smem_u32(&full[i]), 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int bi = blockIdx.x >> 1, r = blockIdx.x & 1;
  const int pos = ctx - 1, QB = pos / 128;
  auto sub_row = [&](int j) { return j == 0 ? 0 : (QB - 7 + j) * 128; };
  const uint64_t pol = policy_evict_last();
  // item code: tile*16 + k (k < 5: K item k; 5..8: V item k-5)
  int order[36], n = 0;
  for (int k = 0; k < 5; ++k) order[n++] = 0 * 16 + k;
  for (int k = 0; k < 5; ++k) order[n++] = 1 * 16 + k;
  for (int i = 0; i < 2; ++i) {
    order[n++] = i * 16 + 5; order[n++] = i * 16 + 6;
    order[n++] = (i + 2) * 16 + 0; order[n++] = (i + 2) * 16 + 1;
    order[n++] = i * 16 + 7; order[n++] = i * 16 + 8;
    for (int k = 2; k < 5; ++k) order[n++] = (i + 2) * 16 + k;
  }
  for (int i = 2; i < 4; ++i) for (int k = 5; k < 9; ++k) order[n++] = i * 16 + k;
  auto issue = [&](int code, int s) {
    const int i = code >> 4, k = code & 15;
    int row, c0, nc;
    if (k < 5) { row = sub_row(2 * i + r); c0 = 2 * k; nc = k < 4 ? 2 : 1; }
    else { const int q = k - 5; row = sub_row(2 * i + (q >> 1)) + 64 * (q & 1); c0 = 4 * r; nc = 2; }
    mbar_arrive_expect_tx(smem_u32(&full[s]), nc * 16384);
    for (int c = 0; c < nc; ++c)
      tma_load_3d(sb + s * 32768 + c * 16384, &map, 64 * (c0 + c), row, bi, smem_u32(&full[s]), pol);
  };
  for (int s = 0; s < S; ++s) issue(order[s], s);
  for (int it = 0; it < n; ++it) {
    const int s = it % S;
    mbar_wait(smem_u32(&full[s]), (it / S) & 1);
    if (it + S < n) issue(order[it + S], s);
  }
}

int main() {
  const size_t bytes = (size_t)B * CTX * 1152;
  void* g;
  cudaMalloc(&g, bytes);
  cudaMemset(g, 1, bytes);
  void* fl;
  cudaMalloc(&fl, 512 << 20);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap map;
  cuuint64_t dims[3] = {576, (cuuint64_t)CTX, (cuuint64_t)B};
  cuuint64_t strides[2] = {1152, (cuuint64_t)1152 * CTX};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto run = [&](auto kern, int S, const char* name) {
    const int smem = S * 32768;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 64; ++i) kern<<<2 * B, 64, smem, st>>>(map, CTX - 2048 * (i % 4));
    cudaStreamEndCapture(st, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemsetAsync(fl, rep, 512 << 20, st);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const double kb = 4.0 * 147456 * 2 * B;  // HBM bytes per step (K once; V re-reads hit L2)
    printf("%-28s ring %2d x 32 KB: %.2f us/step, %.0f GB/s of K rows (err %s)\n", name, S, best * 1e3 / 64,
           kb / (best * 1e-3 / 64) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run(stream<4, false>, 4, "K only");
  run(stream<4, true>, 4, "K + V reload");
  run(stream<6, false>, 6, "K only");
  run(stream<6, true>, 6, "K + V reload");
  run(stream<2, false>, 2, "K only");
  auto run2 = [&](auto kern, int SK, int SV) {
    const int smem = (SK + SV) * 32768;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaGraph_t gr;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 64; ++i) kern<<<2 * B, 96, smem, st>>>(map, CTX - 2048 * (i % 4));
    cudaStreamEndCapture(st, &gr);
    cudaGraphInstantiate(&ge, gr, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemsetAsync(fl, rep, 512 << 20, st);
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("two rings K %d + V %d x 32 KB: %.2f us/step (err %s)\n", SK, SV, best * 1e3 / 64,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(stream3<4>, 4, "interleaved K/V");
  run2(stream2<3, 1>, 3, 1);
  run2(stream2<2, 2>, 2, 2);
  run2(stream2<4, 1>, 4, 1);
  run2(stream2<4, 2>, 4, 2);
  run2(stream2<5, 1>, 5, 1);
  return 0;
}
