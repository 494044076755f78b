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

// 3-D fp32 map {d (contiguous), rows, batch}, box {32, box_rows, 1} (128 B rows), 128B swizzle: the dQ
// epilogue's TMA stores
bool encode_3d_f32(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t batch, int64_t row_stride_el,
                   int64_t batch_stride_el, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc || d % 4 != 0) return false;
  if (rows == 0) rows = 1;
  if (batch == 0) batch = 1;
  cuuint64_t dims[3] = {d, rows, batch};
  cuuint64_t strides[2] = {(cuuint64_t)row_stride_el * 4, (cuuint64_t)(batch_stride_el > 0 ? batch_stride_el : rows * row_stride_el) * 4};
  cuuint32_t box[3] = {32, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 4-D bf16 view {64 (contiguous), rows, d/64 column chunks, batch} of a [batch, rows, d] tensor: one box
// {64, box_rows, box_chunks, 1} fetches box_chunks adjacent 64-column chunks; in SMEM the chunks follow
// each other (box_rows x 128 B each), i.e. the layout of box_chunks separate 3-D loads.
bool encode_4d_chunks(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t batch,
                      int64_t row_stride_el, int64_t batch_stride_el, uint32_t box_rows, uint32_t box_chunks) {
  auto enc = get_encode();
  if (!enc || d % 64 != 0) return false;
  if (rows == 0) rows = 1;
  if (batch == 0) batch = 1;
  cuuint64_t dims[4] = {64, rows, d / 64, batch};
  cuuint64_t strides[3] = {(cuuint64_t)row_stride_el * 2, 128,
                           (cuuint64_t)(batch_stride_el > 0 ? batch_stride_el : rows * row_stride_el) * 2};
  cuuint32_t box[4] = {64, box_rows, box_chunks, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 5-D bf16 view of a per-head tensor [batch, rows, heads, d] (strides in elements): {64, rows, d/64 chunks,
// heads, batch} with box {64, box_rows, box_chunks, 1, 1}: SMEM [chunk][row][64] (SWIZZLE_128B), i.e. the
// layout of box_chunks separate [box_rows x 64] tiles, for one head.
bool encode_5d_heads(CUtensorMap* m, const void* base, uint64_t d, uint64_t rows, uint64_t heads, uint64_t batch,
                     int64_t row_stride_el, int64_t head_stride_el, int64_t batch_stride_el, uint32_t box_rows,
                     uint32_t box_chunks) {
  auto enc = get_encode();
  if (!enc || d % 64 != 0) return false;
  if (rows == 0) rows = 1;
  if (batch == 0) batch = 1;
  cuuint64_t dims[5] = {64, rows, d / 64, heads, batch};
  cuuint64_t strides[4] = {(cuuint64_t)row_stride_el * 2, 128, (cuuint64_t)head_stride_el * 2,
                           (cuuint64_t)batch_stride_el * 2};
  cuuint32_t box[5] = {64, box_rows, box_chunks, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace loza
