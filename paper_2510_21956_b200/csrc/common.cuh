// Shared device helpers for the sm_100a linear-attention kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/la_cuda.h"

namespace lab {

// ---------------------------------------------------------------- dtypes
template <typename T> __device__ __forceinline__ float ld(const T* p);
template <> __device__ __forceinline__ float ld<float>(const float* p) { return __ldg(p); }
template <> __device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(__ldg(p));
}
template <> __device__ __forceinline__ float ld<__half>(const __half* p) {
  return __half2float(__ldg(p));
}
template <typename T> __device__ __forceinline__ T cvt(float x);
template <> __device__ __forceinline__ float cvt<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
template <> __device__ __forceinline__ __half cvt<__half>(float x) { return __float2half_rn(x); }

// Strided (istride, jstride) of a (G, N, D) tensor in a reference layout
// (view.hpp:46-55): FeatureMajor -> (1, N), SequenceMajor -> (D, 1).
struct Strides {
  int64_t is, js;
};
__host__ __device__ inline Strides strides_of(int layout, int64_t n, int64_t d) {
  return layout == LA_FEATURE_MAJOR ? Strides{1, n} : Strides{d, 1};
}

// Degenerate-denominator flag: atomicMin over (group << 32 | position), so the
// lexicographically first offender wins (pool.hpp:36-42 first-item rethrow).
__device__ __forceinline__ void flag_degenerate(unsigned long long* flag, int64_t g, int64_t i) {
  atomicMin(flag, (static_cast<unsigned long long>(g) << 32) | static_cast<unsigned long long>(i));
}

__host__ __device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

constexpr float kEpsF32 = 1e-4f;  // constants.hpp:15-18 (T = float)

}  // namespace lab
