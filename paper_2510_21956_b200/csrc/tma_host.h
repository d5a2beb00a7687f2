// Host-side TMA descriptor construction (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so the library does not link libcuda).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>

namespace lab {

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// Row-major [rows][inner] 16-bit matrix viewed as {64, rows, inner/64} so one box
// {64, box_rows, box_panels} lands in smem as box_panels SW128 panels of
// box_rows x 128 B (the UMMA canonical 128B-swizzled layout).
inline bool make_tma_map(CUtensorMap* m, const void* base, bool bf16, uint64_t rows, uint64_t inner,
                         uint32_t box_rows, uint32_t box_panels) {
  cuuint64_t dims[3] = {64, rows, inner / 64};
  cuuint64_t strides[2] = {inner * 2, 128};
  cuuint32_t box[3] = {64, box_rows, box_panels};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = tma_encode_fn()(
      m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
      const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace lab
