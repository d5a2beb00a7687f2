// Microbenchmark: tcgen05.mma throughput for the shapes the LA kernels use, and
// tcgen05.ld throughput. One CTA per SM, 148 CTAs. Prints cycles per instruction.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../paper_2510_21956_b200/csrc/sm100.cuh"
using namespace lab::sm100;

struct Cfg { int M, N, ts, amn, bmn; const char* name; };

__global__ void __launch_bounds__(256, 1) k_mma(Cfg cfg, int iters, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint64_t* bar = (uint64_t*)(smem + 160 * 1024);
  uint32_t* tslot = (uint32_t*)(bar + 2);
  for (int e = threadIdx.x; e < 160 * 1024 / 16; e += blockDim.x) ((uint4*)smem)[e] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp_id() == 0) tmem_alloc<512>(tslot);
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = *tslot;
  if (warp_id() == 1) {
    const uint32_t id = idesc_f16(cfg.M, cfg.N, 1, cfg.amn, cfg.bmn);
    const uint32_t a = smem_u32(smem), b = a + 64 * 1024;
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t da = cfg.amn ? sdesc_sw128(a + ks * 2048, 16384, 1024) : sdesc_sw128(a + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
          const uint64_t db = cfg.bmn ? sdesc_sw128(b + ks * 2048, 16384, 1024) : sdesc_sw128(b + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
          if (cfg.ts) mma_ts(tm + 256, tm + ks * 8, db, id, 1);
          else mma_ss(tm + 256, da, db, id, 1);
        }
      }
      mma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    unsigned long long t1 = clock64();
    if (lane_id() == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tm);
}

__global__ void __launch_bounds__(128, 1) k_ld(int iters, unsigned long long* out, int wait_each) {
  __shared__ uint32_t tslot;
  if (warp_id() == 0) tmem_alloc<512>(&tslot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tslot + ((warp_id() * 32u) << 16);
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t x[32], y[32];
    tmem_ld32(tm + (it & 7) * 64, x);
    if (wait_each) tmem_ld_wait();
    tmem_ld32(tm + (it & 7) * 64 + 32, y);
    tmem_ld_wait();
#pragma unroll
    for (int u = 0; u < 32; ++u) acc += x[u] ^ y[u];
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345) out[1000] = acc;
  tc_fence_before(); __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tslot);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 2048 * 8);
  unsigned long long h[148];
  const int smem = 160 * 1024 + 2048;
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  Cfg cfgs[] = {{128, 128, 0, 0, 0, "SS M128 N128 K-maj"}, {128, 128, 0, 0, 1, "SS M128 N128 B MN"},
                {128, 256, 0, 0, 0, "SS M128 N256"}, {128, 64, 0, 0, 0, "SS M128 N64"},
                {64, 64, 0, 0, 0, "SS M64 N64"}, {64, 80, 0, 0, 0, "SS M64 N80"}, {64, 128, 0, 0, 0, "SS M64 N128"},
                {128, 16, 0, 1, 0, "SS M128 N16 A MN"}, {128, 64, 1, 0, 0, "TS M128 N64"}, {128, 128, 1, 0, 0, "TS M128 N128"},
                {128, 256, 1, 0, 0, "TS M128 N256"}};
  const int iters = 64;
  for (auto& c : cfgs) {
    for (int grid : {1, 148}) {
      k_mma<<<grid, 256, smem>>>(c, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i]; avg /= grid;
      const double per = avg / (iters * 8);
      const double nominal = (c.M < 128 ? 128 : c.M) * c.N / 256.0;
      printf("%-22s grid %3d: %7.1f cyc/instr (nominal %5.1f) -> %.2f of peak\n", c.name, grid, per, nominal, nominal / per);
    }
  }
  for (int we = 0; we < 2; ++we) {
    k_ld<<<148, 128>>>(1024, d, we);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    const double bytes = 1024.0 * 2 * 32 * 32 * 4 * 4;  // per CTA: iters x 2 loads x (32 lanes x 32 cols x 4B) x 4 warps
    printf("tcgen05.ld 32x32b.x32 (wait_each=%d): %.1f cyc per pair-iter, %.1f B/clk per SM\n", we, avg / 1024, bytes / avg);
  }
  return 0;
}
