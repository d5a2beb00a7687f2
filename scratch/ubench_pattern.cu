// Streaming microbenchmark of the backward sweep's HBM access pattern, without any
// compute: G groups x P segments, one CTA per (segment, group), sweeping C-row chunks
// in reverse. Per chunk it reads Q, K (SequenceMajor: C x 256 B contiguous), V^T, W^T
// (FeatureMajor: 128 rows of 2C bytes at a stride of 2N) and writes dQ (SequenceMajor)
// and dK^T, dV^T (FeatureMajor), like k_bwd_tc. Question: does this pattern alone
// saturate below the copy bandwidth (the sweep measures ~4.7 TB/s)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scratch/ubench_pattern scratch/ubench_pattern.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int C, bool WRITE>
__global__ void __launch_bounds__(512) sweep(const uint4* q, const uint4* k, const uint4* v, const uint4* w,
                                             uint4* dq, uint4* dk, uint4* dv, long N, long seg, uint4* sink) {
  const long g = blockIdx.y, p = blockIdx.x;
  const long s0 = p * seg, nc = seg / C;
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int t = threadIdx.x;
  for (long c = nc - 1; c >= 0; --c) {
    const long row0 = s0 + c * C;
    // SequenceMajor tiles: C rows x 256 B = C * 16 uint4, contiguous
    const long sq = (g * N + row0) * 16;
    for (int e = t; e < C * 16; e += 512) {
      uint4 a = q[sq + e], b = k[sq + e];
      acc.x ^= a.x ^ b.x; acc.y ^= a.y ^ b.y;
      if (WRITE) dq[sq + e] = a;
    }
    // FeatureMajor tiles: 128 feature rows x 2C bytes (C / 8 uint4 each) at stride N
    constexpr int RV = C / 8;
    for (int e = t; e < 128 * RV; e += 512) {
      const long j = e / RV, i = e % RV;
      const long off = (g * 128 + j) * (N / 8) + row0 / 8 + i;
      uint4 a = v[off], b = w[off];
      acc.z ^= a.z ^ b.z; acc.w ^= a.w ^ b.w;
      if (WRITE) {
        dk[off] = a;
        dv[off] = b;
      }
    }
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}

int main() {
  const long G = 64, N = 65536, T = G * N * 128 * 2;
  uint4 *q, *k, *v, *w, *dq, *dk, *dv, *sink;
  cudaMalloc(&q, T); cudaMalloc(&k, T); cudaMalloc(&v, T); cudaMalloc(&w, T);
  cudaMalloc(&dq, T); cudaMalloc(&dk, T); cudaMalloc(&dv, T); cudaMalloc(&sink, 64);
  cudaMemset(q, 1, T); cudaMemset(k, 2, T); cudaMemset(v, 3, T); cudaMemset(w, 4, T);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int P, const char* name, double bytes) {
    const long seg = N / P;
    kern<<<dim3(P, G), 512>>>(q, k, v, w, dq, dk, dv, N, seg, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kern<<<dim3(P, G), 512>>>(q, k, v, w, dq, dk, dv, N, seg, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-34s P=%d  %.3f ms  %.2f TB/s\n", name, P, ms, bytes / ms / 1e9);
  };
  const double rw = 7.0 * T, ro = 4.0 * T;
  for (int P : {2, 4}) {
    run(sweep<64, true>, P, "C=64  read 4 + write 3 tensors", rw);
    run(sweep<128, true>, P, "C=128 read 4 + write 3 tensors", rw);
    run(sweep<64, false>, P, "C=64  read 4 tensors", ro);
    run(sweep<128, false>, P, "C=128 read 4 tensors", ro);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
