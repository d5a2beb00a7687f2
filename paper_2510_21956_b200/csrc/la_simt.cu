#include <cstdlib>
// CUDA-core ("SIMT") linear-attention path: every dtype, D <= 256, any layout.
//
// Same factorisation as the reference CPU kernels (forward_kernels.hpp,
// backward_kernels.hpp) with the sequence split into P segments per group so
// the whole GPU works: (1) per-segment state sums, (2) an exclusive prefix /
// suffix scan across segments, (3) a row sweep per (group, segment) that
// starts from the carried state. Accumulation is fp32. This path serves fp32
// inputs (the <= 1e-5 relative bar needs exact-fp32 arithmetic, not 1xTF32),
// head dims the tensor-core kernels do not instantiate, and non-canonical
// layouts. The bf16/fp16 D=128 hot path is la_sm100.cu.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace lab {

namespace {

constexpr int kTR = 32;   // rows per smem tile in the row sweeps
constexpr int kRB = 128;  // output features per CTA in the row sweeps

// Loads a (rows x D) tile of a strided (G,N,D) tensor into smem as fp32, rows
// [r0, r0+rows) valid, zero elsewhere; coalesced for either layout.
template <typename T>
__device__ __forceinline__ void load_tile(float* dst, int ldd, const T* src, Strides s, int64_t r0,
                                          int rows, int rows_alloc, int64_t D, float scale,
                                          const float* rowscale) {
  const int total = rows_alloc * (int)D;
  const bool fm = s.is == 1;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int li, c;
    if (fm) {
      li = idx % rows_alloc;
      c = idx / rows_alloc;
    } else {
      li = idx / (int)D;
      c = idx % (int)D;
    }
    float x = 0.f;
    if (li < rows) {
      x = ld<T>(src + (r0 + li) * s.is + (int64_t)c * s.js) * scale;
      if (rowscale) x = x / rowscale[li];
    }
    dst[li * ldd + c] = x;
  }
}

// ------------------------------------------------------------------ segment sums
// X[m][j] = sum_rows A_m * B_j ; vA[m] = sum wA * A_m ; vB[j] = sum B_j.
// MODE 0 (KV): A = k, B = v, wA = 1.     (forward S, z, sigma)
// MODE 1 (QW): A = q, B = omega / g, wA = s.  (backward R, u, c)
template <typename T, int MODE>
__global__ void __launch_bounds__(256) k_seg_sums(const T* A, Strides sa, const T* B, Strides sb,
                                                  const float* gvec, const float* svec, int64_t N,
                                                  int64_t D, int64_t seg_len, int P,
                                                  float* states) {
  __shared__ float As[32][33];
  __shared__ float Bs[32][33];
  __shared__ float ws_[32];
  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int tilesj = (int)((D + 31) / 32);
  const int tm = blockIdx.z / tilesj, tj = blockIdx.z % tilesj;
  const int64_t m0 = tm * 32, j0 = tj * 32;
  const int64_t s0 = (int64_t)p * seg_len;
  const int64_t s1 = lmin(N, s0 + seg_len);
  const T* Ag = A + grp * N * D;
  const T* Bg = B + grp * N * D;
  const int ty = threadIdx.x / 8, tx = threadIdx.x % 8;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  float vacc_a = 0.f, vacc_b[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t r0 = s0; r0 < s1; r0 += 32) {
    const int rows = (int)lmin(32, s1 - r0);
    for (int idx = threadIdx.x; idx < 32 * 32; idx += 256) {
      int li, c;
      // A tile: 32 rows x 32 features starting at m0
      if (sa.is == 1) { li = idx % 32; c = idx / 32; } else { li = idx / 32; c = idx % 32; }
      float x = 0.f;
      if (li < rows && m0 + c < D) x = ld<T>(Ag + (r0 + li) * sa.is + (m0 + c) * sa.js);
      As[li][c] = x;
      if (sb.is == 1) { li = idx % 32; c = idx / 32; } else { li = idx / 32; c = idx % 32; }
      float y = 0.f;
      if (li < rows && j0 + c < D) {
        y = ld<T>(Bg + (r0 + li) * sb.is + (j0 + c) * sb.js);
        if (MODE == 1) y = y / gvec[grp * N + r0 + li];
      }
      Bs[li][c] = y;
    }
    if (threadIdx.x < 32) {
      const int li = threadIdx.x;
      ws_[li] = (MODE == 1 && li < rows) ? svec[grp * N + r0 + li] : 1.f;
    }
    __syncthreads();
    for (int li = 0; li < rows; ++li) {
      const float am = As[li][ty];
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] += am * Bs[li][tx * 4 + e];
      if (tx == 0) vacc_a += ws_[li] * am;
      if (ty == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) vacc_b[e] += Bs[li][tx * 4 + e];
      }
    }
    __syncthreads();
  }
  float* st = states + (grp * P + p) * state_floats(D);
  const int64_t m = m0 + ty;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t j = j0 + tx * 4 + e;
    if (m < D && j < D) st[m * D + j] = acc[e];
  }
  if (tj == 0 && tx == 0 && m < D) st[D * D + m] = vacc_a;
  if (tm == 0 && ty == 0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t j = j0 + tx * 4 + e;
      if (j < D) st[D * D + D + j] = vacc_b[e];
    }
  }
  if (blockIdx.z == 0 && threadIdx.x == 0) st[D * D + 2 * D] = (float)(s1 - s0);
}

// ------------------------------------------------------------------ scan
// mode 0: exclusive prefix over segments; 1: exclusive suffix; 2: total in every slot.
__global__ void k_scan_states(float* states, int P, int64_t SZ, const float* carry, int mode) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t grp = blockIdx.y;
  if (e >= SZ) return;
  float* base = states + grp * P * SZ + e;
  float run = carry ? carry[grp * SZ + e] : 0.f;
  if (mode == 0) {
    for (int p = 0; p < P; ++p) {
      const float t = base[p * SZ];
      base[p * SZ] = run;
      run += t;
    }
  } else if (mode == 1) {
    for (int p = P - 1; p >= 0; --p) {
      const float t = base[p * SZ];
      base[p * SZ] = run;
      run += t;
    }
  } else {
    for (int p = 0; p < P; ++p) run += base[p * SZ];
    for (int p = 0; p < P; ++p) base[p * SZ] = run;
  }
}

// Exclusive prefix (suffix) of gathered shard totals for one rank.
__global__ void k_combine(const float* gathered, int nshards, int rank, int suffix, int64_t total,
                          float* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= total) return;
  float run = 0.f;
  if (!suffix) {
    for (int r = 0; r < rank; ++r) run += gathered[r * total + e];
  } else {
    for (int r = nshards - 1; r > rank; --r) run += gathered[r * total + e];
  }
  out[e] = run;
}

// ------------------------------------------------------------------ per-row s_i
// s_i = sum_j o_ij * (omega_ij / g_i)  (backward_kernels.hpp:33-38)
template <typename T>
__global__ void __launch_bounds__(256) k_row_s(const T* o, Strides so, const T* w, Strides sw,
                                               const float* gvec, float* svec, int64_t N,
                                               int64_t D) {
  extern __shared__ float sm[];
  float* ot = sm;                      // [32][D]
  float* wt = sm + 32 * D;             // [32][D]
  const int64_t grp = blockIdx.y;
  const int64_t r0 = blockIdx.x * 32;
  const int rows = (int)lmin(32, N - r0);
  load_tile<T>(ot, (int)D, o + grp * N * D, so, r0, rows, 32, D, 1.f, nullptr);
  load_tile<T>(wt, (int)D, w + grp * N * D, sw, r0, rows, 32, D, 1.f, nullptr);
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int li = warp; li < rows; li += blockDim.x / 32) {
    const float gi = gvec[grp * N + r0 + li];
    float acc = 0.f;
    for (int64_t j = lane; j < D; j += 32) acc += ot[li * D + j] * (wt[li * D + j] / gi);
#pragma unroll
    for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) svec[grp * N + r0 + li] = acc;
  }
}

// ------------------------------------------------------------------ forward rows
// One CTA per (segment, group); thread (j, s) owns state X[j][m] for m in slice s
// (the reference's x2[j][m] = b * S[m][j], forward.hpp:13-18).
template <typename T, int MPT>
__global__ void __launch_bounds__(512) k_fwd_rows(const T* q, Strides sq, const T* k, Strides sk,
                                                   const T* v, Strides sv, T* out, float* gout,
                                                   const float* states, int64_t N, int64_t D,
                                                   int64_t seg_len, int P, float a, float b,
                                                   int causal, int fault, int64_t row_offset,
                                                   int64_t n_total,
                                                   unsigned long long* flag, int nsl) {
  extern __shared__ float sm[];
  const int rb = (int)lmin(D, kRB);  // output features per CTA
  const int TRA = kTR + 1;
  float* qt = sm;                    // [kTR][D]
  float* kt = qt + kTR * D;          // [TRA][D]  (b * k)
  float* vt = kt + TRA * D;          // [TRA][D]
  float* zt = vt + TRA * D;          // [kTR][D]  inclusive b*z per row
  float* ot = zt + kTR * D;          // [kTR][rb]
  float* part = ot + kTR * rb;       // [2][nsl][rb]
  float* zrun = part + 2 * nsl * rb; // [D]
  float* gt = zrun + D;              // [kTR]

  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * seg_len, s1 = lmin(N, s0 + seg_len);
  // blockDim is rounded up to whole warps; threads past nsl*rb only help load
  const bool act = (int)threadIdx.x < nsl * rb;
  const int jl = act ? (int)threadIdx.x % rb : 0, sl = act ? (int)threadIdx.x / rb : nsl;
  const int64_t j0 = (int64_t)blockIdx.z * rb;
  const bool jok = act && j0 + jl < D;
  const int64_t j = jok ? j0 + jl : 0;
  const int64_t SZ = state_floats(D);
  const float* st = states + (grp * P + p) * SZ;
  const T* qg = q + grp * N * D;
  const T* kg = k + grp * N * D;
  const T* vg = v + grp * N * D;

  float X[MPT];
#pragma unroll
  for (int r = 0; r < MPT; ++r) {
    const int64_t m = (int64_t)sl * MPT + r;
    X[r] = (m < D && jok) ? b * st[m * D + j] : 0.f;
  }
  float sigma = jok ? a * st[D * D + D + j] : 0.f;
  for (int64_t m = threadIdx.x; m < D; m += blockDim.x) zrun[m] = b * st[D * D + m];
  const bool offby1 = causal && fault == LA_FAULT_CAUSAL_PREFIX_OFF_BY_ONE;

  for (int64_t r0 = s0; r0 < s1; r0 += kTR) {
    const int rows = (int)lmin(kTR, s1 - r0);
    const int rows_kv = offby1 ? (int)lmin(kTR + 1, N - r0) : rows;
    __syncthreads();
    load_tile<T>(qt, (int)D, qg, sq, r0, rows, kTR, D, 1.f, nullptr);
    load_tile<T>(kt, (int)D, kg, sk, r0, rows_kv, TRA, D, b, nullptr);
    load_tile<T>(vt, (int)D, vg, sv, r0, rows_kv, TRA, D, 1.f, nullptr);
    __syncthreads();
    // running b*z prefix per feature (denominator_causal_core :38-56)
    for (int64_t m = threadIdx.x; m < D; m += blockDim.x) {
      float run = zrun[m];
      for (int li = 0; li < rows; ++li) {
        if (causal) run += kt[li * D + m];
        zt[li * D + m] = run;
      }
      zrun[m] = run;
    }
    __syncthreads();
    {
      const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = (blockDim.x + 31) / 32;
      for (int li = warp; li < rows; li += nw) {
        float acc = 0.f;
        for (int64_t m = lane; m < D; m += 32) acc += qt[li * D + m] * zt[li * D + m];
#pragma unroll
        for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (lane == 0) {
          const int64_t ig = row_offset + r0 + li;
          const float gi = (causal ? a * (float)(ig + 1) : a * (float)n_total) + acc;
          if (fabsf(gi) < kEpsF32) flag_degenerate(flag, grp, ig);
          gt[li] = gi;
        }
      }
    }
    __syncthreads();
    for (int li = 0; li < rows; ++li) {
      const int64_t ig = r0 + li;
      if (causal) {
        if (!offby1) {
          const float vj = vt[li * D + j];
#pragma unroll
          for (int r = 0; r < MPT; ++r) {
            const int64_t m = (int64_t)sl * MPT + r;
            if (m < D) X[r] += kt[li * D + m] * vj;
          }
        } else {
          // CausalPrefixOffByOne (forward_kernels.hpp:86-106): row i sees rows 0..i+1.
          for (int64_t src = (ig == 0 ? 0 : ig + 1); src <= ig + 1 && src < N; ++src) {
            const int ls = (int)(src - r0);
            const float vj = vt[ls * D + j];
#pragma unroll
            for (int r = 0; r < MPT; ++r) {
              const int64_t m = (int64_t)sl * MPT + r;
              if (m < D) X[r] += kt[ls * D + m] * vj;
            }
          }
        }
      }
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < MPT; ++r) {
        const int64_t m = (int64_t)sl * MPT + r;
        if (m < D) acc += qt[li * D + m] * X[r];
      }
      if (act) part[((li & 1) * nsl + sl) * rb + jl] = acc;
      __syncthreads();
      if (act && sl == 0) {
        if (causal) sigma += a * vt[li * D + j];
        float f = sigma;
        for (int s = 0; s < nsl; ++s) f += part[((li & 1) * nsl + s) * rb + jl];
        ot[li * rb + jl] = f / gt[li];
      }
    }
    __syncthreads();
    // FeatureMajor output out[g][j][i]: i fastest for coalescing.
    T* og = out + grp * N * D;
    for (int idx = threadIdx.x; idx < rows * rb; idx += blockDim.x) {
      const int li = idx % rows, c = idx / rows;
      if (j0 + c < D) og[(j0 + c) * N + r0 + li] = cvt<T>(ot[li * rb + c]);
    }
    if (blockIdx.z == 0)
      for (int li = threadIdx.x; li < rows; li += blockDim.x) gout[grp * N + r0 + li] = gt[li];
  }
}

// ------------------------------------------------------------------ backward rows
// Thread (r, s) owns X[r][c] for c in slice s and produces out_r per row.
//   MODE 0 dQ  (prefix): A=b*k, B=v, C=w_hat ; vec += A ;      out = dot - s*vec
//   MODE 1 dK  (suffix): A=b*q, B=w_hat, C=v ; vec += s*A ;    out = dot -/+ vec
//   MODE 2 dV  (suffix): A=w_hat, B=b*q, C=k ; vec += a*A ;    out = vec + dot
// (grad_q_causal_core :21-57, grad_k_alpha_core :61-91 + grad_k_beta_core :95-130,
//  grad_v_causal_core :134-168; the *_full_core variants when !causal.)
template <typename T, int MPT, int MODE>
__global__ void __launch_bounds__(512) k_bwd_rows(const T* q, Strides sq, const T* k, Strides sk,
                                                   const T* v, Strides sv, const T* w, Strides sw,
                                                   const float* gvec, const float* svec, T* outp,
                                                   Strides so, const float* states, int64_t N,
                                                   int64_t D, int64_t seg_len, int P, float a,
                                                   float b, int causal, int fault, int nsl) {
  extern __shared__ float sm[];
  const int rb = (int)lmin(D, kRB);
  float* At = sm;               // [kTR][D]
  float* Bt = At + kTR * D;     // [kTR][D]
  float* Ct = Bt + kTR * D;     // [kTR][D]
  float* ot = Ct + kTR * D;     // [kTR][rb]
  float* part = ot + kTR * rb;  // [2][nsl][rb]
  float* gt = part + 2 * nsl * rb;  // [kTR]
  float* stile = gt + kTR;          // [kTR]

  const int p = blockIdx.x;
  const int64_t grp = blockIdx.y;
  const int64_t s0 = (int64_t)p * seg_len, s1 = lmin(N, s0 + seg_len);
  const bool act = (int)threadIdx.x < nsl * rb;
  const int rl = act ? (int)threadIdx.x % rb : 0, sl = act ? (int)threadIdx.x / rb : nsl;
  const int64_t r0b = (int64_t)blockIdx.z * rb;
  const bool rok = act && r0b + rl < D;
  const int r = rok ? (int)(r0b + rl) : 0;
  const int64_t SZ = state_floats(D);
  const float* st = states + (grp * P + p) * SZ;
  const int64_t off = grp * N * D;

  float X[MPT];
  float vec = 0.f;
#pragma unroll
  for (int cc = 0; cc < MPT; ++cc) {
    const int64_t c = (int64_t)sl * MPT + cc;
    float x = 0.f;
    if (c < D && rok) x = MODE == 2 ? st[c * D + r] : st[(int64_t)r * D + c];
    X[cc] = b * x;
  }
  if (MODE == 0) vec = b * st[D * D + r];      // b*z prefix
  if (MODE == 1) vec = b * st[D * D + r];      // b*u suffix
  if (MODE == 2) vec = a * st[D * D + D + r];  // a*c suffix
  const bool flip = fault == LA_FAULT_FLIP_BETA_K_SIGN;
  const bool drop = fault == LA_FAULT_DROP_GRAD_V_CONSTANT_TERM;

  const int64_t ntiles = (s1 - s0 + kTR - 1) / kTR;
  for (int64_t tt = 0; tt < ntiles; ++tt) {
    const int64_t tile = MODE == 0 ? tt : ntiles - 1 - tt;
    const int64_t r0 = s0 + tile * kTR;
    const int rows = (int)lmin(kTR, s1 - r0);
    __syncthreads();
    for (int li = threadIdx.x; li < kTR; li += blockDim.x) {
      gt[li] = li < rows ? gvec[grp * N + r0 + li] : 1.f;
      stile[li] = li < rows ? svec[grp * N + r0 + li] : 0.f;
    }
    __syncthreads();
    if (MODE == 0) {
      load_tile<T>(At, (int)D, k + off, sk, r0, rows, kTR, D, b, nullptr);
      load_tile<T>(Bt, (int)D, v + off, sv, r0, rows, kTR, D, 1.f, nullptr);
      load_tile<T>(Ct, (int)D, w + off, sw, r0, rows, kTR, D, 1.f, gt);
    } else if (MODE == 1) {
      load_tile<T>(At, (int)D, q + off, sq, r0, rows, kTR, D, b, nullptr);
      load_tile<T>(Bt, (int)D, w + off, sw, r0, rows, kTR, D, 1.f, gt);
      load_tile<T>(Ct, (int)D, v + off, sv, r0, rows, kTR, D, 1.f, nullptr);
    } else {
      load_tile<T>(At, (int)D, w + off, sw, r0, rows, kTR, D, 1.f, gt);
      load_tile<T>(Bt, (int)D, q + off, sq, r0, rows, kTR, D, b, nullptr);
      load_tile<T>(Ct, (int)D, k + off, sk, r0, rows, kTR, D, 1.f, nullptr);
    }
    __syncthreads();
    for (int step = 0; step < rows; ++step) {
      const int li = MODE == 0 ? step : rows - 1 - step;
      const float ar = At[li * D + r];
      if (causal) {
#pragma unroll
        for (int cc = 0; cc < MPT; ++cc) {
          const int64_t c = (int64_t)sl * MPT + cc;
          if (c < D) X[cc] += ar * Bt[li * D + c];
        }
      }
      float acc = 0.f;
#pragma unroll
      for (int cc = 0; cc < MPT; ++cc) {
        const int64_t c = (int64_t)sl * MPT + cc;
        if (c < D) acc += X[cc] * Ct[li * D + c];
      }
      if (act) part[((step & 1) * nsl + sl) * rb + rl] = acc;
      __syncthreads();
      if (act && sl == 0) {
        float dot = 0.f;
        for (int s = 0; s < nsl; ++s) dot += part[((step & 1) * nsl + s) * rb + rl];
        float res;
        if (MODE == 0) {
          if (causal) vec += ar;
          res = dot - stile[li] * vec;
        } else if (MODE == 1) {
          if (causal) vec += stile[li] * ar;
          res = flip ? dot + vec : dot - vec;
        } else {
          if (causal) vec += a * ar;
          res = drop ? dot : vec + dot;
        }
        ot[li * rb + rl] = res;
      }
    }
    __syncthreads();
    T* og = outp + off;
    const bool fm = so.is == 1;
    for (int idx = threadIdx.x; idx < rows * rb; idx += blockDim.x) {
      int li, c;
      if (fm) { li = idx % rows; c = idx / rows; } else { li = idx / rb; c = idx % rb; }
      if (r0b + c < D) og[(r0 + li) * so.is + (r0b + c) * so.js] = cvt<T>(ot[li * rb + c]);
    }
  }
}

// Non-causal backward: the reference's full cores take sums over all rows
// *without* the b factor inside the state for the dV constant (grad_v_full_core
// alpha_v = a * sum w_hat). The row kernel above handles that through vec.

template <typename T> struct Dt;

int mpt_for(int64_t D) { return D <= 128 ? 32 : 64; }
int nsl_for(int64_t D) { return (int)((D + mpt_for(D) - 1) / mpt_for(D)); }

int64_t rb_for(int64_t D) { return lmin(D, kRB); }
size_t fwd_rows_smem(int64_t D, int nsl) {
  const int64_t rb = rb_for(D);
  return sizeof(float) * (size_t)(kTR * D + 2 * (kTR + 1) * D + kTR * D + kTR * rb + 2 * nsl * rb + D + kTR);
}
size_t bwd_rows_smem(int64_t D, int nsl) {
  const int64_t rb = rb_for(D);
  return sizeof(float) * (size_t)(3 * kTR * D + kTR * rb + 2 * nsl * rb + 2 * kTR);
}

template <typename T>
cudaError_t forward_t(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  const int64_t G = L.G, N = L.N, D = L.D;
  const int P = simt_segments(G, N, L.fault);
  const int64_t seg = (N + P - 1) / P;
  const int64_t SZ = state_floats(D);
  float* states = ws.base;
  const Strides sq = strides_of(t.lq, N, D), sk = strides_of(t.lk, N, D),
                sv = strides_of(t.lv, N, D);
  const int tiles = (int)(((D + 31) / 32) * ((D + 31) / 32));
  {
    ProfScope ps_("k_seg_sums", L.stream);
    k_seg_sums<T, 0><<<dim3(P, G, tiles), 256, 0, L.stream>>>(
      (const T*)t.k, sk, (const T*)t.v, sv, nullptr, nullptr, N, D, seg, P, states);
  }
  {
    ProfScope ps_("k_scan_states", L.stream);
    k_scan_states<<<dim3((SZ + 255) / 256, G), 256, 0, L.stream>>>(states, P, SZ, L.carry_prefix,
                                                                 L.causal ? 0 : 2);
  }
  note_launch(2);
  const int nsl = nsl_for(D);
  const int threads = (int)((nsl * rb_for(D) + 31) / 32 * 32);
  const int nrb = (int)((D + rb_for(D) - 1) / rb_for(D));
  const size_t smem = fwd_rows_smem(D, nsl);
  const int64_t ntot = L.n_total > 0 ? L.n_total : N;
  if (mpt_for(D) == 32) {
    auto kern = k_fwd_rows<T, 32>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    {
      ProfScope ps_("k_fwd_rows", L.stream);
      kern<<<dim3(P, G, nrb), threads, smem, L.stream>>>(
        (const T*)t.q, sq, (const T*)t.k, sk, (const T*)t.v, sv, (T*)out, g, states, N, D, seg,
        P, L.a, L.b, L.causal, L.fault, L.row_offset, ntot, ws.flag, nsl);
    }
  } else {
    auto kern = k_fwd_rows<T, 64>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    {
      ProfScope ps_("k_fwd_rows", L.stream);
      kern<<<dim3(P, G, nrb), threads, smem, L.stream>>>(
        (const T*)t.q, sq, (const T*)t.k, sk, (const T*)t.v, sv, (T*)out, g, states, N, D, seg,
        P, L.a, L.b, L.causal, L.fault, L.row_offset, ntot, ws.flag, nsl);
    }
  }
  note_launch(1);
  return cudaGetLastError();
}

template <typename T, int MPT, int MODE>
void launch_bwd_rows(const Launch& L, const Tensors& t, const float* svec, void* outp, int lout,
                     const float* states, int P, int64_t seg) {
  const int64_t N = L.N, D = L.D;
  const int nsl = nsl_for(D);
  const size_t smem = bwd_rows_smem(D, nsl);
  auto kern = k_bwd_rows<T, MPT, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nrb = (int)((D + rb_for(D) - 1) / rb_for(D));
  {
    ProfScope ps_(MODE == 0 ? "k_bwd_rows_dq" : MODE == 1 ? "k_bwd_rows_dk" : "k_bwd_rows_dv", L.stream);
    kern<<<dim3(P, L.G, nrb), (int)((nsl * rb_for(D) + 31) / 32 * 32), smem, L.stream>>>(
      (const T*)t.q, strides_of(t.lq, N, D), (const T*)t.k, strides_of(t.lk, N, D),
      (const T*)t.v, strides_of(t.lv, N, D), (const T*)t.w, strides_of(t.lw, N, D), t.g, svec,
      (T*)outp, strides_of(lout, N, D), states, N, D, seg, P, L.a, L.b, L.causal, L.fault, nsl);
  }
  note_launch(1);
}

template <typename T>
void prep_row_s(int64_t D) {
  cudaFuncSetAttribute(k_row_s<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(sizeof(float) * 64 * D));
}

template <typename T>
cudaError_t backward_t(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv,
                       Workspace ws) {
  const int64_t G = L.G, N = L.N, D = L.D;
  const int P = simt_segments(G, N, L.fault);
  const int64_t seg = (N + P - 1) / P;
  const int64_t SZ = state_floats(D);
  float* svec = ws.base;
  float* statesS = svec + G * N;
  float* statesR = statesS + G * P * SZ;
  const Strides sq = strides_of(t.lq, N, D), sk = strides_of(t.lk, N, D),
                sv = strides_of(t.lv, N, D), so = strides_of(t.lo, N, D),
                sw = strides_of(t.lw, N, D);
  prep_row_s<T>(D);
  {
    ProfScope ps_("k_row_s", L.stream);
    k_row_s<T><<<dim3((N + 31) / 32, G), 256, sizeof(float) * 64 * D, L.stream>>>(
      (const T*)t.o, so, (const T*)t.w, sw, t.g, svec, N, D);
  }
  const int tiles = (int)(((D + 31) / 32) * ((D + 31) / 32));
  {
    ProfScope ps_("k_seg_sums", L.stream);
    k_seg_sums<T, 0><<<dim3(P, G, tiles), 256, 0, L.stream>>>((const T*)t.k, sk, (const T*)t.v, sv,
                                                            nullptr, nullptr, N, D, seg, P,
                                                            statesS);
  }
  {
    ProfScope ps_("k_seg_sums", L.stream);
    k_seg_sums<T, 1><<<dim3(P, G, tiles), 256, 0, L.stream>>>((const T*)t.q, sq, (const T*)t.w, sw,
                                                            t.g, svec, N, D, seg, P, statesR);
  }
  {
    ProfScope ps_("k_scan_states", L.stream);
    k_scan_states<<<dim3((SZ + 255) / 256, G), 256, 0, L.stream>>>(statesS, P, SZ, L.carry_prefix,
                                                                 L.causal ? 0 : 2);
  }
  {
    ProfScope ps_("k_scan_states", L.stream);
    k_scan_states<<<dim3((SZ + 255) / 256, G), 256, 0, L.stream>>>(statesR, P, SZ, L.carry_suffix,
                                                                 L.causal ? 1 : 2);
  }
  note_launch(5);
  if (mpt_for(D) == 32) {
    launch_bwd_rows<T, 32, 0>(L, t, svec, dq, LA_SEQUENCE_MAJOR, statesS, P, seg);
    launch_bwd_rows<T, 32, 1>(L, t, svec, dk, LA_FEATURE_MAJOR, statesR, P, seg);
    launch_bwd_rows<T, 32, 2>(L, t, svec, dv, LA_FEATURE_MAJOR, statesR, P, seg);
  } else {
    launch_bwd_rows<T, 64, 0>(L, t, svec, dq, LA_SEQUENCE_MAJOR, statesS, P, seg);
    launch_bwd_rows<T, 64, 1>(L, t, svec, dk, LA_FEATURE_MAJOR, statesR, P, seg);
    launch_bwd_rows<T, 64, 2>(L, t, svec, dv, LA_FEATURE_MAJOR, statesR, P, seg);
  }
  return cudaGetLastError();
}

}  // namespace

int simt_segments(int64_t G, int64_t N, int fault) {
  if (fault != LA_FAULT_NONE) return 1;  // fault variants are defined on the unsplit sweep
  int64_t want = (2 * 148 + G - 1) / G;
  const int e = tuning().simt_seg_rows;  // measurement override of the minimum segment
  const int64_t min_rows = e > 0 ? e : 32;  // config 1 (G=4, N=2048): 1.93 -> 0.46 ms vs 256
  int64_t cap = (N + min_rows - 1) / min_rows;
  return (int)std::max<int64_t>(1, std::min(want, cap));
}

size_t simt_forward_ws_floats(int64_t G, int64_t N, int64_t D, int fault) {
  return (size_t)(G * simt_segments(G, N, fault) * state_floats(D));
}
size_t simt_backward_ws_floats(int64_t G, int64_t N, int64_t D, int fault) {
  return (size_t)(G * N + 2 * G * simt_segments(G, N, fault) * state_floats(D));
}

cudaError_t simt_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws) {
  switch (L.dtype) {
    case LA_F32: return forward_t<float>(L, t, out, g, ws);
    case LA_BF16: return forward_t<__nv_bfloat16>(L, t, out, g, ws);
    case LA_F16: return forward_t<__half>(L, t, out, g, ws);
  }
  return cudaErrorInvalidValue;
}

cudaError_t simt_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv,
                          Workspace ws) {
  switch (L.dtype) {
    case LA_F32: return backward_t<float>(L, t, dq, dk, dv, ws);
    case LA_BF16: return backward_t<__nv_bfloat16>(L, t, dq, dk, dv, ws);
    case LA_F16: return backward_t<__half>(L, t, dq, dk, dv, ws);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
static cudaError_t fwd_shard_state_t(const Launch& L, const Tensors& t, float* out) {
  const int64_t N = L.N, D = L.D;
  const int tiles = (int)(((D + 31) / 32) * ((D + 31) / 32));
  {
    ProfScope ps_("k_seg_sums", L.stream);
    k_seg_sums<T, 0><<<dim3(1, L.G, tiles), 256, 0, L.stream>>>(
      (const T*)t.k, strides_of(t.lk, N, D), (const T*)t.v, strides_of(t.lv, N, D), nullptr,
      nullptr, N, D, N, 1, out);
  }
  note_launch(1);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t bwd_shard_state_t(const Launch& L, const Tensors& t, float* out, Workspace ws) {
  const int64_t N = L.N, D = L.D;
  float* svec = ws.base;
  prep_row_s<T>(D);
  {
    ProfScope ps_("k_row_s", L.stream);
    k_row_s<T><<<dim3((N + 31) / 32, L.G), 256, sizeof(float) * 64 * D, L.stream>>>(
      (const T*)t.o, strides_of(t.lo, N, D), (const T*)t.w, strides_of(t.lw, N, D), t.g, svec, N,
      D);
  }
  const int tiles = (int)(((D + 31) / 32) * ((D + 31) / 32));
  {
    ProfScope ps_("k_seg_sums", L.stream);
    k_seg_sums<T, 1><<<dim3(1, L.G, tiles), 256, 0, L.stream>>>(
      (const T*)t.q, strides_of(t.lq, N, D), (const T*)t.w, strides_of(t.lw, N, D), t.g, svec, N,
      D, N, 1, out);
  }
  note_launch(2);
  return cudaGetLastError();
}

cudaError_t simt_forward_shard_state(const Launch& L, const Tensors& t, float* state_out) {
  switch (L.dtype) {
    case LA_F32: return fwd_shard_state_t<float>(L, t, state_out);
    case LA_BF16: return fwd_shard_state_t<__nv_bfloat16>(L, t, state_out);
    case LA_F16: return fwd_shard_state_t<__half>(L, t, state_out);
  }
  return cudaErrorInvalidValue;
}

cudaError_t simt_backward_shard_state(const Launch& L, const Tensors& t, float* state_out,
                                      Workspace ws) {
  switch (L.dtype) {
    case LA_F32: return bwd_shard_state_t<float>(L, t, state_out, ws);
    case LA_BF16: return bwd_shard_state_t<__nv_bfloat16>(L, t, state_out, ws);
    case LA_F16: return bwd_shard_state_t<__half>(L, t, state_out, ws);
  }
  return cudaErrorInvalidValue;
}

cudaError_t combine_shard_states(int64_t G, int64_t D, const float* gathered, int nshards,
                                 int rank, int suffix, float* carry_out, cudaStream_t s) {
  const int64_t total = G * state_floats(D);
  {
    ProfScope ps_("k_combine", s);
    k_combine<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(gathered, nshards, rank, suffix, total,
                                                           carry_out);
  }
  note_launch(1);
  return cudaGetLastError();
}

}  // namespace lab
