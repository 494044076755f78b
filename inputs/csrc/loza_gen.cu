// Seeded counter-based synthetic input generator, device side.
//
// CUDA twin of inputs/gen.py (same integer / IEEE-fp32 recipe, element by
// element; tests/test_gen_gpu.py checks the two bitwise). Holds none of the
// method's arithmetic; it exists so that multi-GB inputs (a 2.4 GB Q at 32K,
// a 77 GB cache at 1M) are written directly into HBM while the host regenerates
// any row it needs for the oracle.
//
// C ABI (no torch types):
//   int loza_gen_fill(void* dst, const loza_gen_spec_t* spec,
//                     int64_t row_start, int64_t row_count, cudaStream_t s)
//     dst       device pointer to row_count contiguous rows of spec->d elements
//               (bf16 bits or fp32), i.e. rows [row_start, row_start+row_count)
//               of the flat [batch*n*heads, d] view of the logical tensor
//     returns   0 on success, 1 on invalid spec, 4 on CUDA launch error
#include <cuda_runtime.h>
#include <stdint.h>

extern "C" {
typedef struct {
  uint64_t seed;
  int32_t tensor_id;
  int32_t dtype;      // 0 = f32, 1 = bf16
  int64_t batch, n, heads, d;
  int32_t kind;       // 0 plain, 1 kv_marker, 2 kv_sink, 3 q_sink
  int32_t block;      // b (kv_marker)
  int32_t marker_mod; // d_v (kv_marker)
  int32_t col;        // coordinate (kv_sink / q_sink)
  int64_t sink_rows;  // positions boosted by kv_sink
  float amp;
} loza_gen_spec_t;
}

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kTidMul = 0xD1B54A32D192ED03ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen_kernel(void* __restrict__ dst, loza_gen_spec_t spec, uint64_t key,
                           int64_t row_start, int64_t count) {
  const float kScale = __uint_as_float(0x37DDB3D7u);  // fp32(sqrt(3)/65536)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int64_t row_local = i / spec.d;
    const int64_t col = i - row_local * spec.d;
    const int64_t row = row_start + row_local;
    const uint64_t idx = (uint64_t)(row * spec.d + col);
    const uint64_t bits = mix64(key + (idx + 1ull) * kGolden);
    const int64_t s = (int64_t)(bits & 0xFFFFull) + (int64_t)((bits >> 16) & 0xFFFFull) +
                      (int64_t)((bits >> 32) & 0xFFFFull) + (int64_t)(bits >> 48);
    float z = __fmul_rn((float)(s - 131070), kScale);
    if (spec.kind != 0) {
      const int64_t pos = (row / spec.heads) % spec.n;
      bool hit;
      if (spec.kind == 1)      hit = col == (pos / spec.block) % spec.marker_mod;
      else if (spec.kind == 2) hit = (col == spec.col) && (pos < spec.sink_rows);
      else                     hit = (col == spec.col);
      if (hit) z = __fadd_rn(z, spec.amp);
    }
    if (spec.dtype == 1) {
      uint32_t u = __float_as_uint(z);
      u = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
      reinterpret_cast<uint16_t*>(dst)[i] = (uint16_t)u;
    } else {
      reinterpret_cast<float*>(dst)[i] = z;
    }
  }
}

}  // namespace

extern "C" int loza_gen_fill(void* dst, const loza_gen_spec_t* spec, int64_t row_start,
                             int64_t row_count, cudaStream_t stream) {
  if (!spec || (!dst && row_count > 0) || spec->d <= 0 || spec->heads <= 0 || spec->n <= 0 ||
      row_start < 0 || row_count < 0 || (spec->kind == 1 && (spec->block <= 0 || spec->marker_mod <= 0)))
    return 1;
  if (row_count == 0) return 0;
  const uint64_t key = mix64((spec->seed * kGolden) ^ ((uint64_t)(uint32_t)spec->tensor_id * kTidMul));
  const int64_t count = row_count * spec->d;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  gen_kernel<<<(unsigned)blocks, 256, 0, stream>>>(dst, *spec, key, row_start, count);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
