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

namespace lab {
// In-kernel carry combine (replaces a separate scan launch): the CTA's threads
// [tid, nthr) write dst[e] = (base ? base[e] : 0) + sum_{q in [q0, q1)} recs[q * SZ + e].
__device__ __forceinline__ void combine_records(float* dst, const float* base, const float* recs, int q0,
                                                int q1, int64_t SZ, int tid, int nthr) {
  // 4 float4 positions per thread and pass, 2 records per step: 8 independent loads in
  // flight (the records are L2 / HBM resident; a serial chain would be latency-bound)
  constexpr int kU = 4;
  const int64_t step = 4 * (int64_t)nthr;
  for (int64_t e0 = 4 * tid; e0 < SZ; e0 += kU * step) {
    float4 acc[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t e = e0 + u * step;
      acc[u] = (base && e < SZ) ? *(const float4*)(base + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    int q = q0;
    for (; q + 1 < q1; q += 2) {
      float4 v[2][kU];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int64_t e = e0 + u * step;
          v[h][u] = e < SZ ? *(const float4*)(recs + (q + h) * SZ + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          acc[u].x += v[h][u].x; acc[u].y += v[h][u].y; acc[u].z += v[h][u].z; acc[u].w += v[h][u].w;
        }
    }
    if (q < q1) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t e = e0 + u * step;
        if (e < SZ) {
          const float4 v = *(const float4*)(recs + q * SZ + e);
          acc[u].x += v.x; acc[u].y += v.y; acc[u].z += v.z; acc[u].w += v.w;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t e = e0 + u * step;
      if (e < SZ) *(float4*)(dst + e) = acc[u];
    }
  }
}
}  // namespace lab
