// tcgen05.mma throughput per shape with compile-time, fully unrolled issue loops.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../paper_2510_21956_b200/csrc/sm100.cuh"
using namespace lab::sm100;

template <int M, int N, int TS, int AMN, int BMN>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
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
    constexpr uint32_t id = idesc_f16(M, N, 1, AMN, BMN);
    const uint32_t a = smem_u32(smem), b = a + 64 * 1024;
    uint64_t da[8], db[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      da[ks] = AMN ? sdesc_sw128(a + ks * 2048, 16384, 1024) : sdesc_sw128(a + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
      db[ks] = BMN ? sdesc_sw128(b + ks * 2048, 16384, 1024) : sdesc_sw128(b + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
    }
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          if (TS) mma_ts(tm + 256, tm + ks * 8, db[ks], id, 1);
          else mma_ss(tm + 256, da[ks], db[ks], id, 1);
        }
      }
      mma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    if (lane_id() == 0) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tm);
}

template <int M, int N, int TS, int AMN, int BMN>
void run(const char* name, unsigned long long* d) {
  const int smem = 160 * 1024 + 2048, iters = 64;
  cudaFuncSetAttribute(k<M, N, TS, AMN, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<M, N, TS, AMN, BMN><<<148, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
  const double per = avg / (iters * 8), nominal = (M < 128 ? 128 : M) * N / 256.0;
  const double bytes = (TS ? 0 : M * 32) + N * 32;
  printf("%-24s %6.1f cyc/instr (nominal %5.1f, %.2f) smem %.0f B/clk\n", name, per, nominal, nominal / per, bytes / per);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 2048 * 8);
  run<128, 128, 0, 0, 0>("SS M128 N128", d);
  run<128, 128, 0, 1, 1>("SS M128 N128 A,B MN", d);
  run<128, 256, 0, 0, 0>("SS M128 N256", d);
  run<128, 64, 0, 0, 0>("SS M128 N64", d);
  run<128, 16, 0, 1, 0>("SS M128 N16 A MN", d);
  run<64, 64, 0, 0, 0>("SS M64 N64", d);
  run<64, 80, 0, 0, 0>("SS M64 N80", d);
  run<64, 128, 0, 0, 0>("SS M64 N128", d);
  run<64, 64, 0, 1, 1>("SS M64 N64 A,B MN", d);
  run<128, 64, 1, 0, 0>("TS M128 N64", d);
  run<128, 128, 1, 0, 0>("TS M128 N128", d);
  run<128, 256, 1, 0, 0>("TS M128 N256", d);
  return 0;
}
