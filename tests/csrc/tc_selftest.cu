// Hardware self-test of the sm_100a building blocks used by la_sm100.cu:
// UMMA smem descriptors (K-major / MN-major, 128B swizzle), A-from-TMEM,
// TMEM ld/st, commit -> mbarrier, and TMA 3D loads. One CTA computes
// D[128x128] = A[128xK] * B[128xK]^T (K = 128) and writes D in fp32.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "../../paper_2510_21956_b200/csrc/sm100.cuh"

using namespace lab::sm100;

__global__ void __launch_bounds__(128) k_selftest(const __nv_bfloat16* A, const __nv_bfloat16* B,
                                                  float* D, int mode,
                                                  const __grid_constant__ CUtensorMap tmA,
                                                  const __grid_constant__ CUtensorMap tmB) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;              // 32 KB
  uint8_t* sB = smem + 32768;      // 32 KB
  uint64_t* bar = (uint64_t*)(smem + 65536);
  uint32_t* tslot = (uint32_t*)(smem + 65536 + 64);
  const int tid = threadIdx.x;
  const int M = 128, N = 128, K = 128;
  const bool a_mn = mode == 1, b_mn = mode == 2, a_tmem = mode == 3, use_tma = mode == 4;
  if (mode >= 5) {
    // M = N = 64, K = 128: A rows m < 64, B rows n < 64
    const bool amn = mode == 6;
    if (warp_id() == 0) tmem_alloc<512>(tslot);
    if (tid == 0) {
      mbar_init(&bar[0], 1);
      fence_barrier_init();
    }
    for (int e = tid; e < 64 * K; e += 128) {
      const int m = e / K, k = e % K;
      const uint32_t offa = amn ? sw128_off(k, m, K) : sw128_off(m, k, 64);
      *(__nv_bfloat16*)(sA + offa) = A[e];
      *(__nv_bfloat16*)(sB + sw128_off(m, k, 64)) = B[e];
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *tslot;
    const uint32_t dlane = mode == 5 ? (16u << 16) : 0u;
    if (warp_id() == 1) {
      if (elect_one()) {
        const uint32_t id = idesc_f16(64, 64, 1, amn ? 1 : 0, 0, mode == 6 ? 1 : 0);
        for (int s = 0; s < K / 16; ++s) {
          const uint64_t da = amn ? sdesc_sw128(smem_u32(sA) + s * 2048, K * 128, 1024)
                                  : sdesc_sw128(smem_u32(sA) + (s / 4) * 64 * 128 + (s % 4) * 32, 16, 1024);
          const uint64_t db = sdesc_sw128(smem_u32(sB) + (s / 4) * 64 * 128 + (s % 4) * 32, 16, 1024);
          mma_ss(tb + dlane, da, db, id, s > 0);
        }
        mma_commit(&bar[0]);
      }
      __syncwarp();
    }
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    // row m of the M=64 accumulator lives in lane (m % 16) + 32 * (m / 16) (+16 for the upper half)
    const uint32_t qd = warp_id() % 4, l = lane_id();
    uint32_t r[32];
    for (int c0 = 0; c0 < 64; c0 += 32) {
      tmem_ld32(tb + ((qd * 32u) << 16) + c0, r);
      tmem_ld_wait();
      const bool mine = mode == 5 ? l >= 16 : l < 16;
      const int row = (int)(qd * 16 + (l & 15));
      if (mine)
        for (int c = 0; c < 32; ++c) D[row * 128 + c0 + c] = __uint_as_float(r[c]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp_id() == 0) tmem_dealloc<512>(tb);
    return;
  }

  if (warp_id() == 0) tmem_alloc<512>(tslot);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (use_tma) {
    if (tid == 0) {
      mbar_expect_tx(&bar[1], 65536);
      tma_load_3d(sA, &tmA, &bar[1], 0, 0, 0);
      tma_load_3d(sB, &tmB, &bar[1], 0, 0, 0);
    }
    mbar_wait(&bar[1], 0);
  } else {
    for (int e = tid; e < M * K; e += 128) {
      const int m = e / K, k = e % K;
      __nv_bfloat16 x = A[e];
      if (!a_tmem) {
        const uint32_t off = a_mn ? sw128_off(k, m, K) : sw128_off(m, k, M);
        *(__nv_bfloat16*)(sA + off) = x;
      }
      const int n = m;
      __nv_bfloat16 y = B[n * K + k];
      const uint32_t offb = b_mn ? sw128_off(k, n, K) : sw128_off(n, k, N);
      *(__nv_bfloat16*)(sB + offb) = y;
    }
    if (a_tmem) {
      // lane m holds A row m, 16-bit pairs packed per 32-bit column, at columns [256, 320)
      const int m = (warp_id() % 4) * 32 + lane_id();
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t r[32];
        for (int c = 0; c < 32; ++c) {
          const int k = 2 * (c0 + c);
          r[c] = pack_bf16(__bfloat162float(A[m * K + k]), __bfloat162float(A[m * K + k + 1]));
        }
        tmem_st32(tbase + ((uint32_t)(warp_id() % 4) * 32u << 16) + 256 + c0, r);
      }
      tmem_st_wait();
    }
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp_id() == 1) {
    if (elect_one()) {
      const uint32_t id = idesc_f16(M, N, 1, a_mn ? 1 : 0, b_mn ? 1 : 0);
      for (int s = 0; s < K / 16; ++s) {
        uint64_t da, db;
        if (a_mn)
          da = sdesc_sw128(smem_u32(sA) + s * 2048, K * 128, 1024);
        else
          da = sdesc_sw128(smem_u32(sA) + (s / 4) * M * 128 + (s % 4) * 32, 16, 1024);
        if (b_mn)
          db = sdesc_sw128(smem_u32(sB) + s * 2048, K * 128, 1024);
        else
          db = sdesc_sw128(smem_u32(sB) + (s / 4) * N * 128 + (s % 4) * 32, 16, 1024);
        if (a_tmem)
          mma_ts(tbase, tbase + 256 + s * 8, db, id, s > 0);
        else
          mma_ss(tbase, da, db, id, s > 0);
      }
      mma_commit(&bar[0]);
    }
    __syncwarp();
  }
  mbar_wait(&bar[0], 0);
  tc_fence_after();
  const int m = (warp_id() % 4) * 32 + lane_id();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tbase + ((uint32_t)(warp_id() % 4) * 32u << 16) + c0, r);
    tmem_ld_wait();
    for (int c = 0; c < 32; ++c) D[m * N + c0 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tbase);
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

// [rows][128] bf16 row-major -> smem [2 panels][rows][64] SW128
static CUtensorMap map_rows128(const void* base, int rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {128 * 2, 128};  // bytes for dims 1, 2
  cuuint32_t box[3] = {64, (cuuint32_t)rows, 2};
  cuuint32_t es[3] = {1, 1, 1};
  get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

extern "C" int tc_selftest(const void* A, const void* B, float* D, int mode) {
  CUtensorMap ta = map_rows128(A, 128), tb = map_rows128(B, 128);
  const int smem = 65536 + 1024 + 256;
  cudaFuncSetAttribute(k_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_selftest<<<1, 128, smem>>>((const __nv_bfloat16*)A, (const __nv_bfloat16*)B, D, mode, ta, tb);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
