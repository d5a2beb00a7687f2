// tcgen05.ld throughput/latency alone and while SS/TS MMAs (M128 N128, accumulating in
// TMEM columns [256, 384)) run. Warps 4..7 load TMEM columns [0, 128).
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../paper_2510_21956_b200/csrc/sm100.cuh"
using namespace lab::sm100;

__global__ void __launch_bounds__(256, 1) k(int mma_iters, int ts, int ld_iters, unsigned long long* out) {
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
    uint64_t da[8], db[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      da[ks] = sdesc_sw128(a + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
      db[ks] = sdesc_sw128(b + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
    }
    unsigned long long t0 = clock64();
    if (mma_iters > 0) {
      if (elect_one()) {
        for (int it = 0; it < mma_iters; ++it) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            if (ts) mma_ts(tm + 256, tm + 128 + ks * 8, db[ks], id, 1);
            else mma_ss(tm + 256, da[ks], db[ks], id, 1);
          }
        }
        mma_commit(bar);
      }
      __syncwarp();
      mbar_wait(bar, 0);
    }
    if (lane_id() == 0) out[blockIdx.x * 2] = clock64() - t0;
  } else if (warp_id() >= 4) {
    const uint32_t base = tm + (((warp_id() & 3) * 32u) << 16);
    uint32_t acc = 0;
    unsigned long long t0 = clock64();
    for (int it = 0; it < ld_iters; ++it) {
      uint32_t x[32], y[32];
      tmem_ld32(base + (it & 1) * 64, x);
      tmem_ld32(base + (it & 1) * 64 + 32, y);
      tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 32; ++u) acc += x[u] ^ y[u];
    }
    if (threadIdx.x == 128) out[blockIdx.x * 2 + 1] = clock64() - t0;
    if (acc == 12345) out[5000] = acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8192 * 8);
  unsigned long long h[2 * 148];
  const int smem = 160 * 1024 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int cfg[5][3] = {{0, 0, 256}, {64, 0, 0}, {64, 0, 256}, {64, 1, 0}, {64, 1, 256}};
  for (auto& c : cfg) {
    k<<<148, 256, smem>>>(c[0], c[1], c[2], d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0, l = 0;
    for (int i = 0; i < 148; ++i) { m += h[2 * i]; l += h[2 * i + 1]; }
    m /= 148; l /= 148;
    printf("mma_iters=%d ts=%d ld_iters=%d: mma %.0f cyc (%.1f/instr), ld %.0f cyc (%.1f cyc per 8KB-per-warp iter, %.0f B/clk)\n",
           c[0], c[1], c[2], m, c[0] ? m / (c[0] * 8) : 0.0, l, c[2] ? l / c[2] : 0.0, c[2] ? c[2] * 32768.0 / l : 0.0);
  }
  return 0;
}
