// Non-causal (forward_full / backward_full) path for head dimensions other than 128:
// every contraction of the unmasked algebra is a plain batched GEMM over the groups
// (cuBLAS, bf16/fp16 operands, fp32 accumulation), joined by small streaming kernels.
// forward_kernels.hpp:133-206 / backward_kernels.hpp:173-288, per group (row-major):
//   S = K^T V, z = sum k, sigma = sum v
//   g_i = a N + b q_i . z;  O = (a sigma + b Q S) / g  computed as  O^T = S~^T Q~^T with
//     S~ = [b S ; a sigma^T ; 0] and Q~ = [q_i / g_i , 1 / g_i , 0]  (the division folded in)
//   w_hat = omega / g, s_i = o_i . w_hat_i, R = Q^T W_hat, u = sum s q, c = sum w_hat
//   dQ = [W_hat | s] [(b S)^T ; -b z^T]          (the rank-1 term folded in)
//   dK^T = (b R) V^T - b u 1^T,  dV^T = (b R)^T K^T + a c 1^T
// The D = 128 case runs the tcgen05 kernels (la_sm100*.cu); this path replaces the
// CUDA-core sweep for D = 256 and the zero-padding detour for D < 128.
#include <cublas_v2.h>

#include "common.cuh"
#include "internal.h"

namespace lab {
namespace {

cublasHandle_t handle() {
  static thread_local cublasHandle_t h = nullptr;
  if (!h) cublasCreate(&h);
  return h;
}

// Row-major C[M x N] = op(A) op(B), batched over groups (cuBLAS is column-major:
// a row-major X is the column-major X^T, so C^T = op(B)^T op(A)^T).
cublasStatus_t rm_gemm(cudaStream_t st, bool ta, bool tb, int M, int N, int K, const void* A, int lda,
                       long long sA, cudaDataType tA, const void* B, int ldb, long long sB, cudaDataType tB,
                       void* C, int ldc, long long sC, cudaDataType tC, int batch, float alpha = 1.f,
                       float beta = 0.f) {
  cublasHandle_t h = handle();
  cublasSetStream(h, st);
  return cublasGemmStridedBatchedEx(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, N, M, K,
                                    &alpha, B, tB, ldb, sB, A, tA, lda, sA, &beta, C, tC, ldc, sC, batch,
                                    CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
}

constexpr int kChunk = 256;  // rows per partial column sum

// partial[g][c][m] = sum over rows [c*kChunk, ...) of x[g][n][m] (* w[g][n]); x SequenceMajor.
// A thread owns 8 consecutive features (one 16-byte load per row); the D/8 threads of
// a row and the 256/(D/8) row lanes are reduced through shared memory.
template <typename T>
__global__ void __launch_bounds__(256) k_colsum_part(const T* x, const float* w, float* part, int64_t N, int D,
                                                     int nchunk) {
  __shared__ float red[2048];  // [lanes][D], lanes * D <= 2048
  const int64_t g = blockIdx.y;
  const int c = blockIdx.x;
  const int C8 = D / 8, lanes = 256 / C8;
  const int m8 = threadIdx.x % C8, rl = threadIdx.x / C8;
  const int64_t n0 = (int64_t)c * kChunk, n1 = lmin(N, n0 + kChunk);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (rl < lanes)
    for (int64_t n = n0 + rl; n < n1; n += lanes) {
      const uint4 u = __ldg((const uint4*)(x + (g * N + n) * D) + m8);
      const T* e = (const T*)&u;
      const float wn = w ? w[g * N + n] : 1.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += (float)e[k] * wn;
    }
  __syncthreads();
  float* r = red;  // [lanes][D]
  if (rl < lanes)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[rl * D + 8 * m8 + k] = acc[k];
  __syncthreads();
  for (int m = threadIdx.x; m < D; m += blockDim.x) {
    float t = 0.f;
    for (int l = 0; l < lanes; ++l) t += r[l * D + m];
    part[((int64_t)g * nchunk + c) * D + m] = t;
  }
}
// out[g][m] = sum_c partial[g][c][m]; one thread per (g, m), 256-wide blocks over G * D.
__global__ void k_sum_part(const float* part, float* out, int nchunk, int D, int64_t GD) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= GD) return;
  const int64_t g = e / D;
  const int m = (int)(e % D);
  float acc = 0.f;
  for (int c = 0; c < nchunk; ++c) acc += part[((int64_t)g * nchunk + c) * D + m];
  out[e] = acc;
}

// out[g][j] = sum_i y[g][j][i] (FeatureMajor rows of N, row stride rs, N % 8 == 0),
// one CTA per (j, g), 16-byte loads.
template <typename T>
__global__ void __launch_bounds__(256) k_rowsum(const T* y, float* out, int64_t N, int D, int64_t rs,
                                                int64_t gstride) {
  __shared__ float red[8];
  const int64_t g = blockIdx.y;
  const int j = blockIdx.x;
  const uint4* row = (const uint4*)(y + g * gstride + (int64_t)j * rs);
  float acc = 0.f;
  for (int64_t i = threadIdx.x; i < N / 8; i += blockDim.x) {
    const uint4 u = __ldg(row + i);
    const T* e = (const T*)&u;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += (float)e[k];
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[g * D + j] = t;
  }
}

// g_i = a n_total + b q_i . z and Q~ = [q_i / g_i, 1 / g_i, 0...] (Dp = D + 8 columns):
// 8 lanes per row, 16-byte loads / stores (4 rows per warp instruction).
template <typename T>
__global__ void __launch_bounds__(256) k_qtilde(const T* q, const float* z, float a, float b, float n_total,
                                                T* qt, float* gout, int64_t rows, int64_t N, int D, int Dp,
                                                unsigned long long* flag) {
  const int64_t r = (int64_t)blockIdx.x * 32 + threadIdx.x / 8;
  const int l8 = threadIdx.x % 8;
  const bool ok = r < rows;
  const int64_t rr = ok ? r : 0;
  const int64_t g = rr / N;
  const uint4* qr = (const uint4*)(q + rr * D);
  const float* zg = z + g * D;
  const int C8 = D / 8;
  float dot = 0.f;
  for (int c = l8; c < C8; c += 8) {
    const uint4 u = __ldg(qr + c);
    const T* e = (const T*)&u;
#pragma unroll
    for (int k = 0; k < 8; ++k) dot += (float)e[k] * zg[8 * c + k];
  }
  dot += __shfl_xor_sync(0xffffffffu, dot, 1);
  dot += __shfl_xor_sync(0xffffffffu, dot, 2);
  dot += __shfl_xor_sync(0xffffffffu, dot, 4);
  if (!ok) return;
  const float gi = a * n_total + b * dot;
  if (l8 == 0) {
    gout[r] = gi;
    if (fabsf(gi) < kEpsF32) flag_degenerate(flag, g, r - g * N);
  }
  const float inv = 1.f / gi;
  uint4* o = (uint4*)(qt + r * Dp);
  for (int c = l8; c <= C8; c += 8) {
    uint4 u = make_uint4(0, 0, 0, 0);
    T* e = (T*)&u;
    if (c < C8) {
      const uint4 v = __ldg(qr + c);
      const T* ev = (const T*)&v;
#pragma unroll
      for (int k = 0; k < 8; ++k) e[k] = cvt<T>((float)ev[k] * inv);
    } else {
      e[0] = cvt<T>(inv);
    }
    o[c] = u;
  }
}

// S~ [Dp][D] = [b S ; a sigma ; 0] and (bwd) T_S [Dp][D] = [(b S)^T ; -b z ; 0], bR = b R.
template <typename T>
__global__ void k_pack_state(const float* S, int64_t sgs, const float* vec, int64_t vgs, float row_scale,
                             float vec_scale, int transpose, T* out, int D, int Dp) {
  const int64_t g = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)Dp * D) return;
  const int r = (int)(e / D), col = (int)(e % D);
  float v = 0.f;
  if (r < D) v = row_scale * (transpose ? S[g * sgs + (int64_t)col * D + r] : S[g * sgs + (int64_t)r * D + col]);
  else if (r == D && vec) v = vec_scale * vec[g * vgs + col];
  out[g * Dp * D + e] = cvt<T>(v);
}

// Saved-state record per group: [S (D x D) | z | sigma | count | 0 padding].
__global__ void k_write_records(const float* S, const float* z, const float* sig, float count, float* rec, int D) {
  const int64_t g = blockIdx.y;
  const int64_t SZ = state_floats(D);
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= SZ) return;
  const int64_t DD = (int64_t)D * D;
  float v = 0.f;
  if (e < DD) v = S[g * DD + e];
  else if (e < DD + D) v = z[g * D + (e - DD)];
  else if (e < DD + 2 * D) v = sig[g * D + (e - DD - D)];
  else if (e == DD + 2 * D) v = count;
  rec[g * SZ + e] = v;
}

// w_hat^T [Dp][N] = [omega^T / g ; s ; 0] and s_i = sum_j o_ij w_hat_ij (fp32): a thread
// owns 8 consecutive rows i (16-byte FeatureMajor loads / stores along i).
template <typename T>
__global__ void __launch_bounds__(256) k_what(const T* w, const T* o, const float* gv, T* wt, float* s, int64_t N,
                                              int D, int Dp) {
  const int64_t i8 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const int64_t g = blockIdx.y;
  if (i8 >= N) return;
  float ginv[8], si[8];
  {
    const float4 g0 = *(const float4*)(gv + g * N + i8), g1 = *(const float4*)(gv + g * N + i8 + 4);
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ginv[k] = gg[k];
      si[k] = 0.f;
    }
  }
  const T* wg = w + g * N * D + i8;
  const T* og = o + g * N * D + i8;
  T* dst = wt + g * (int64_t)Dp * N + i8;
  for (int j = 0; j < D; ++j) {
    const uint4 wu = __ldg((const uint4*)(wg + (int64_t)j * N)), ou = __ldg((const uint4*)(og + (int64_t)j * N));
    const T* we = (const T*)&wu;
    const T* oe = (const T*)&ou;
    uint4 r;
    T* re = (T*)&r;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float wh = (float)we[k] / ginv[k];
      re[k] = cvt<T>(wh);
      si[k] += (float)oe[k] * wh;
    }
    *(uint4*)(dst + (int64_t)j * N) = r;
  }
  uint4 r;
  T* re = (T*)&r;
#pragma unroll
  for (int k = 0; k < 8; ++k) re[k] = cvt<T>(si[k]);
  *(uint4*)(dst + (int64_t)D * N) = r;
  *(float4*)(s + g * N + i8) = make_float4(si[0], si[1], si[2], si[3]);
  *(float4*)(s + g * N + i8 + 4) = make_float4(si[4], si[5], si[6], si[7]);
  const uint4 zero = make_uint4(0, 0, 0, 0);
  for (int j = D + 1; j < Dp; ++j) *(uint4*)(dst + (int64_t)j * N) = zero;
}

// y[g][j][i] += scale * vec[g][j] (FeatureMajor, in place): 8 values per thread
// (16-byte accesses), grid (row blocks, j, g) so no index division.
template <typename T>
__global__ void __launch_bounds__(256) k_add_rowbias(T* y, const float* vec, float scale, int64_t N, int D) {
  const int64_t g = blockIdx.z;
  const int j = blockIdx.y;
  const int64_t i8 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i8 >= N) return;
  const float add = scale * vec[g * D + j];
  uint4* p = (uint4*)(y + (g * D + j) * N + i8);
  uint4 u = *p;
  T* e = (T*)&u;
#pragma unroll
  for (int k = 0; k < 8; ++k) e[k] = cvt<T>((float)e[k] + add);
  *p = u;
}

struct Scratch {
  char* base = nullptr;
  size_t off = 0;
  template <typename X>
  X* take(size_t n) {
    X* p = (X*)(base + off);
    off += (n * sizeof(X) + 255) & ~(size_t)255;
    return p;
  }
};

template <typename T>
cudaError_t fwd_t(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  const int64_t G = L.G, N = L.N;
  const int D = (int)L.D, Dp = D + 8;
  const cudaDataType dt = L.dtype == LA_BF16 ? CUDA_R_16BF : CUDA_R_16F;
  const int nchunk = (int)((N + kChunk - 1) / kChunk);
  cudaStream_t st = L.stream;
  keep_pool_memory();
  size_t bytes = 0;
  bytes += ((size_t)G * D * D * 4 + 255) & ~255ull;           // S
  bytes += ((size_t)G * nchunk * D * 4 + 255) & ~255ull;      // partial sums
  bytes += 2 * (((size_t)G * D * 4 + 255) & ~255ull);         // z, sigma
  bytes += ((size_t)G * Dp * D * sizeof(T) + 255) & ~255ull;  // S~
  bytes += ((size_t)G * N * Dp * sizeof(T) + 255) & ~255ull;  // Q~
  Scratch sc;
  cudaError_t e = cudaMallocAsync((void**)&sc.base, bytes, st);
  if (e != cudaSuccess) return e;
  float* S = sc.take<float>((size_t)G * D * D);
  float* part = sc.take<float>((size_t)G * nchunk * D);
  float* z = sc.take<float>((size_t)G * D);
  float* sig = sc.take<float>((size_t)G * D);
  T* St = sc.take<T>((size_t)G * Dp * D);
  T* Qt = sc.take<T>((size_t)G * N * Dp);
  const T* q = (const T*)t.q;
  const T* k = (const T*)t.k;
  const T* v = (const T*)t.v;
  int launches = 0;
  cublasStatus_t cs = rm_gemm(st, true, true, D, D, (int)N, k, D, N * D, dt, v, (int)N, N * D, dt, S, D,
                              (long long)D * D, CUDA_R_32F, (int)G);  // S = K^T V
  k_colsum_part<T><<<dim3(nchunk, (unsigned)G), 256, 0, st>>>(k, nullptr, part, N, D, nchunk);
  k_sum_part<<<(unsigned)((G * D + 255) / 256), 256, 0, st>>>(part, z, nchunk, D, G * D);
  k_rowsum<T><<<dim3(D, (unsigned)G), 256, 0, st>>>(v, sig, N, D, N, N * D);
  k_qtilde<T><<<(unsigned)((G * N + 31) / 32), 256, 0, st>>>(q, z, L.a, L.b, (float)L.n_total, Qt, g, G * N, N, D,
                                                            Dp, ws.flag);
  k_pack_state<T><<<dim3((unsigned)((Dp * D + 255) / 256), (unsigned)G), 256, 0, st>>>(S, (int64_t)D * D, sig, D, L.b,
                                                                                     L.a, 0, St, D, Dp);
  if (L.saved_out) {  // the K/V totals as state records for the backward (header P = -1)
    write_saved_header(L.saved_out, (double)G, (double)N, (double)D, -1, 0, st);
    const int64_t SZ = state_floats(D);
    k_write_records<<<dim3((unsigned)((SZ + 255) / 256), (unsigned)G), 256, 0, st>>>(S, z, sig, (float)N,
                                                                                     L.saved_out + kSavedHeader, D);
  }
  if (cs == CUBLAS_STATUS_SUCCESS)  // O^T = S~^T Q~^T  (FeatureMajor)
    cs = rm_gemm(st, true, true, D, (int)N, Dp, St, D, (long long)Dp * D, dt, Qt, Dp, N * Dp, dt, out, (int)N,
                 N * D, dt, (int)G);
  launches += 8;
  note_launch(launches);
  cudaFreeAsync(sc.base, st);
  if (cs != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  return cudaGetLastError();
}

template <typename T>
cudaError_t bwd_t(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv) {
  const int64_t G = L.G, N = L.N;
  const int D = (int)L.D, Dp = D + 8;
  const cudaDataType dt = L.dtype == LA_BF16 ? CUDA_R_16BF : CUDA_R_16F;
  const int nchunk = (int)((N + kChunk - 1) / kChunk);
  cudaStream_t st = L.stream;
  const float a = L.a, b = L.b;
  keep_pool_memory();
  size_t bytes = 0;
  bytes += 2 * (((size_t)G * D * D * 4 + 255) & ~255ull);       // S, R
  bytes += ((size_t)G * nchunk * D * 4 + 255) & ~255ull;         // partial sums
  bytes += 3 * (((size_t)G * D * 4 + 255) & ~255ull);            // z, u, c
  bytes += ((size_t)G * N * 4 + 255) & ~255ull;                  // s
  bytes += ((size_t)G * Dp * D * sizeof(T) + 255) & ~255ull;     // T_S
  bytes += ((size_t)G * D * D * sizeof(T) + 255) & ~255ull;      // bR
  bytes += ((size_t)G * Dp * N * sizeof(T) + 255) & ~255ull;     // [W_hat^T ; s]
  Scratch sc;
  cudaError_t e = cudaMallocAsync((void**)&sc.base, bytes, st);
  if (e != cudaSuccess) return e;
  float* S = sc.take<float>((size_t)G * D * D);
  float* R = sc.take<float>((size_t)G * D * D);
  float* part = sc.take<float>((size_t)G * nchunk * D);
  float* z = sc.take<float>((size_t)G * D);
  float* u = sc.take<float>((size_t)G * D);
  float* c = sc.take<float>((size_t)G * D);
  float* s = sc.take<float>((size_t)G * N);
  T* TS = sc.take<T>((size_t)G * Dp * D);
  T* bR = sc.take<T>((size_t)G * D * D);
  T* Wt = sc.take<T>((size_t)G * Dp * N);
  const T* q = (const T*)t.q;
  const T* k = (const T*)t.k;
  const T* v = (const T*)t.v;
  const T* o = (const T*)t.o;
  const T* w = (const T*)t.w;
  // S, z: the forward's saved totals (la_forward_save) or recomputed from K, V
  const float* Sp = S;
  const float* zp = z;
  int64_t sgs = (int64_t)D * D;
  cublasStatus_t cs = CUBLAS_STATUS_SUCCESS;
  if (L.saved_in) {
    sgs = state_floats(D);
    Sp = L.saved_in + kSavedHeader;
    zp = Sp + (int64_t)D * D;
  } else {
    cs = rm_gemm(st, true, true, D, D, (int)N, k, D, N * D, dt, v, (int)N, N * D, dt, S, D, (long long)D * D,
                 CUDA_R_32F, (int)G);  // S = K^T V
    k_colsum_part<T><<<dim3(nchunk, (unsigned)G), 256, 0, st>>>(k, nullptr, part, N, D, nchunk);
    k_sum_part<<<(unsigned)((G * D + 255) / 256), 256, 0, st>>>(part, z, nchunk, D, G * D);
  }
  k_what<T><<<dim3((unsigned)((N / 8 + 255) / 256), (unsigned)G), 256, 0, st>>>(w, o, t.g, Wt, s, N, D, Dp);
  k_colsum_part<T><<<dim3(nchunk, (unsigned)G), 256, 0, st>>>(q, s, part, N, D, nchunk);
  k_sum_part<<<(unsigned)((G * D + 255) / 256), 256, 0, st>>>(part, u, nchunk, D, G * D);                                     // u = Q^T s
  k_rowsum<T><<<dim3(D, (unsigned)G), 256, 0, st>>>(Wt, c, N, D, N, (int64_t)Dp * N);             // c
  if (cs == CUBLAS_STATUS_SUCCESS)  // R = Q^T W_hat
    cs = rm_gemm(st, true, true, D, D, (int)N, q, D, N * D, dt, Wt, (int)N, (long long)Dp * N, dt, R, D,
                 (long long)D * D, CUDA_R_32F, (int)G);
  const dim3 pg((unsigned)((Dp * D + 255) / 256), (unsigned)G);
  k_pack_state<T><<<pg, 256, 0, st>>>(Sp, sgs, zp, sgs == (int64_t)D * D ? D : sgs, b, -b, 1, TS, D, Dp);  // [(b S)^T ; -b z]
  k_pack_state<T><<<dim3((unsigned)((D * D + 255) / 256), (unsigned)G), 256, 0, st>>>(R, (int64_t)D * D, nullptr, 0, b,
                                                                                   0.f, 0, bR, D, D);
  if (cs == CUBLAS_STATUS_SUCCESS)  // dQ = [W_hat | s] T_S  (SequenceMajor)
    cs = rm_gemm(st, true, false, (int)N, D, Dp, Wt, (int)N, (long long)Dp * N, dt, TS, D, (long long)Dp * D, dt,
                 dq, D, N * D, dt, (int)G);
  if (cs == CUBLAS_STATUS_SUCCESS)  // dK^T = (b R) V^T
    cs = rm_gemm(st, false, false, D, (int)N, D, bR, D, (long long)D * D, dt, v, (int)N, N * D, dt, dk, (int)N,
                 N * D, dt, (int)G);
  if (cs == CUBLAS_STATUS_SUCCESS)  // dV^T = (b R)^T K^T
    cs = rm_gemm(st, true, true, D, (int)N, D, bR, D, (long long)D * D, dt, k, D, N * D, dt, dv, (int)N, N * D, dt,
                 (int)G);
  const dim3 bg((unsigned)((N / 8 + 255) / 256), (unsigned)D, (unsigned)G);
  k_add_rowbias<T><<<bg, 256, 0, st>>>((T*)dk, u, -b, N, D);
  k_add_rowbias<T><<<bg, 256, 0, st>>>((T*)dv, c, a, N, D);
  note_launch(14);
  cudaFreeAsync(sc.base, st);
  if (cs != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  return cudaGetLastError();
}

}  // namespace

bool gemm_full_supported(const Launch& L, const Tensors& t) {
  return !L.causal && (L.dtype == LA_BF16 || L.dtype == LA_F16) && L.D != 128 && L.D % 8 == 0 && L.D <= 256 &&
         L.fault == LA_FAULT_NONE && L.carry_prefix == nullptr && L.carry_suffix == nullptr && L.row_offset == 0 &&
         L.N % 8 == 0 && t.lq == LA_SEQUENCE_MAJOR && t.lk == LA_SEQUENCE_MAJOR && t.lv == LA_FEATURE_MAJOR &&
         (t.o == nullptr || t.lo == LA_FEATURE_MAJOR) && (t.w == nullptr || t.lw == LA_FEATURE_MAJOR) &&
         L.G * L.N * (L.D + 8) < (1ll << 31);
}

cudaError_t gemm_forward_full(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  ProfScope ps("la_gemm_fwd_full", L.stream);
  return L.dtype == LA_BF16 ? fwd_t<__nv_bfloat16>(L, t, out, g, ws) : fwd_t<__half>(L, t, out, g, ws);
}

cudaError_t gemm_backward_full(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv) {
  ProfScope ps("la_gemm_bwd_full", L.stream);
  return L.dtype == LA_BF16 ? bwd_t<__nv_bfloat16>(L, t, dq, dk, dv) : bwd_t<__half>(L, t, dq, dk, dv);
}

}  // namespace lab
