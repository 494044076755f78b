// Host-side TMA descriptor encoding (driver entry point, no libcuda link).
#include <cudaTypedefs.h>

#include "internal.h"

namespace loza {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }();
  return fn;
}

// 3-D bf16 map {d (contiguous), rows, batch}, box {64, box_rows, 1}, 128B swizzle
}  // namespace

bool encode_3d(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t batch, int64_t row_stride_el,
               int64_t batch_stride_el, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  if (rows == 0) rows = 1;
  if (batch == 0) batch = 1;
  cuuint64_t dims[3] = {d, rows, batch};
  cuuint64_t strides[2] = {(cuuint64_t)row_stride_el * 2, (cuuint64_t)(batch_stride_el > 0 ? batch_stride_el : rows * row_stride_el) * 2};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}


}  // namespace loza
