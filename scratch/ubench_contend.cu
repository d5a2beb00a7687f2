// Does a stream of SS tcgen05.mma starve LSU shared-memory traffic (and vice versa)?
// warp 1 issues `mma_iters` x 8 SS MMAs (M128 N128) over smem [0, 128K); warps 4..7 run an
// LDS.128 loop over smem [128K, 160K). Reports cycles for each side, alone and together.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include "../paper_2510_21956_b200/csrc/sm100.cuh"
using namespace lab::sm100;

__global__ void __launch_bounds__(256, 1) k(int mma_iters, int lds_iters, int sts, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* bar = (uint64_t*)(smem + 160 * 1024);
  uint32_t* tslot = (uint32_t*)(bar + 2);
  for (int e = threadIdx.x; e < 160 * 1024 / 16; e += blockDim.x) ((uint4*)smem)[e] = make_uint4(e, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp_id() == 0) tmem_alloc<512>(tslot);
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = *tslot;
  if (warp_id() == 1) {
    const uint32_t id = idesc_f16(128, 128, 1, 0, 0);
    const uint32_t a = smem_u32(smem), b = a + 64 * 1024;
    unsigned long long t0 = clock64();
    if (mma_iters > 0) {
      if (elect_one()) {
        for (int it = 0; it < mma_iters; ++it)
          for (int ks = 0; ks < 8; ++ks)
            mma_ss(tm, sdesc_sw128(a + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024),
                   sdesc_sw128(b + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024), id, 1);
        mma_commit(bar);
      }
      __syncwarp();
      mbar_wait(bar, 0);
    }
    if (lane_id() == 0) out[blockIdx.x * 2] = clock64() - t0;
  } else if (warp_id() >= 4) {
    const int t = threadIdx.x - 128;
    uint8_t* base = smem + 128 * 1024;
    uint4 acc = make_uint4(0, 0, 0, 0);
    unsigned long long t0 = clock64();
    for (int it = 0; it < lds_iters; ++it) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint4* pp = (uint4*)(base + ((t * 16 + u * 2048 + it * 16) & 32767));
        if (sts) *pp = acc;
        else {
          const uint4 v = *pp;
          acc.x ^= v.x; acc.y += v.y;
        }
      }
    }
    __syncwarp();
    if (t == 0) out[blockIdx.x * 2 + 1] = clock64() - t0;
    if (acc.x == 0x12345) out[5000] = acc.y;
  }
  tc_fence_before(); __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8192 * 8);
  unsigned long long h[2 * 148];
  const int smem = 160 * 1024 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int sts = 0; sts < 2; ++sts) {
    int cfg[3][2] = {{64, 0}, {0, 256}, {64, 256}};
    for (auto& c : cfg) {
      k<<<148, 256, smem>>>(c[0], c[1], sts, d);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double m = 0, l = 0;
      for (int i = 0; i < 148; ++i) { m += h[2 * i]; l += h[2 * i + 1]; }
      m /= 148; l /= 148;
      const double lds_bytes = (double)c[1] * 8 * 128 * 16;
      printf("%s mma_iters=%d lds_iters=%d: mma %.0f cyc (%.1f per instr), lsu %.0f cyc (%.1f B/clk)\n",
             sts ? "STS" : "LDS", c[0], c[1], m, c[0] ? m / (c[0] * 8) : 0.0, l, c[1] ? lds_bytes / l : 0.0);
    }
  }
  return 0;
}
