// Input prologue and diagnostic entry points around the hot path (SURVEY §8(f)
// rows 3-4), on the CUDA cores: all of them are O(N·D) streaming passes or
// O(N·D²) per-row sweeps that the reference exposes as separate API calls.
//
//   la_normalize_qk        normalize_qk        plan.cpp:95-117
//   la_relayout            relayout            tensor.cpp:101-119
//   la_make_omega_hat      make_omega_hat      backward.cpp:74-91
//   la_constant_term_pass  constant_term_pass  forward.cpp:97-107  (constant_causal_core :22-34)
//   la_linear_term_pass    linear_term_pass    forward.cpp:109-131 (linear_causal_core :63-128, g_vec = null)
//   la_alpha_term_pass     alpha_term_pass     backward.cpp:103-128 (grad_k_alpha_core :61-91, unit g)
//   la_beta_term_pass      beta_term_pass      backward.cpp:130-153 (grad_k_beta_core :95-130, unit g)
//
// Term accumulators are the reference's TermAccumulator (forward.hpp:44-50):
// FeatureMajor G·N·D, here fp32 on the device.
#include <cstdio>
#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace lab {
namespace {

// ------------------------------------------------------------------ normalize_qk
// SequenceMajor: one warp per row (contiguous D values).
template <typename T>
__global__ void __launch_bounds__(256) k_normalize_seq(const T* x, T* y, int64_t rows, int D) {
  const int64_t row = (int64_t)blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  const T* xr = x + row * D;
  float sq = 0.f;
  for (int j = lane; j < D; j += 32) {
    const float v = ld(xr + j);
    sq += v * v;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
  const float inv = sq == 0.f ? 1.f : 1.f / sqrtf(sq);  // zero rows (padding) stay zero
  T* yr = y + row * D;
  for (int j = lane; j < D; j += 32) yr[j] = cvt<T>(ld(xr + j) * inv);
}

// FeatureMajor: one thread per row; consecutive threads read consecutive rows of a
// feature column, so every pass over j is coalesced.
template <typename T>
__global__ void __launch_bounds__(256) k_normalize_feat(const T* x, T* y, int64_t G, int64_t N, int D) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = blockIdx.y;
  if (i >= N) return;
  const T* xg = x + g * N * D + i;
  float sq = 0.f;
  for (int j = 0; j < D; ++j) {
    const float v = ld(xg + (int64_t)j * N);
    sq += v * v;
  }
  const float inv = sq == 0.f ? 1.f : 1.f / sqrtf(sq);
  T* yg = y + g * N * D + i;
  for (int j = 0; j < D; ++j) yg[(int64_t)j * N] = cvt<T>(ld(xg + (int64_t)j * N) * inv);
}

// ------------------------------------------------------------------ relayout (+ / g)
// 32 x 32 (row, feature) tiles through shared memory; loads and stores are each
// coalesced along whichever index is contiguous in their layout. With `rowdiv`
// every value of row i is divided by rowdiv[g*N + i] (make_omega_hat).
template <typename T>
__global__ void __launch_bounds__(256) k_relayout(const T* x, int lx, T* y, int ly, int64_t N, int64_t D,
                                                  const float* rowdiv) {
  __shared__ float tile[32][33];  // [feature][row]
  const int64_t g = blockIdx.z, i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const T* xg = x + g * N * D;
  for (int r = ty; r < 32; r += 8) {
    // FeatureMajor source: tx walks rows (contiguous); SequenceMajor: tx walks features
    const int64_t i = lx == LA_FEATURE_MAJOR ? i0 + tx : i0 + r;
    const int64_t j = lx == LA_FEATURE_MAJOR ? j0 + r : j0 + tx;
    float v = 0.f;
    if (i < N && j < D) {
      v = ld(xg + (lx == LA_FEATURE_MAJOR ? j * N + i : i * D + j));
      if (rowdiv) v = v / rowdiv[g * N + i];
    }
    tile[j - j0][i - i0] = v;
  }
  __syncthreads();
  T* yg = y + g * N * D;
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = ly == LA_FEATURE_MAJOR ? i0 + tx : i0 + r;
    const int64_t j = ly == LA_FEATURE_MAJOR ? j0 + r : j0 + tx;
    if (i < N && j < D) yg[ly == LA_FEATURE_MAJOR ? j * N + i : i * D + j] = cvt<T>(tile[j - j0][i - i0]);
  }
}

// ------------------------------------------------------------------ term sweeps
// One generic causal sweep covers the four term passes. Per group, rows in
// prefix (ascending) or suffix (descending) order:
//   X[o][c] += U_t[o] * W_t[c]        (the running D x D state of the reference core)
//   out_t[o] = sum_c X[o][c] * Y_t[c]
// written into the FeatureMajor fp32 accumulator acc[g][o][t] by assign / add / subtract.
//   constant  o = j, Dc = 1, U = a*v, W = 1, Y = 1                     prefix, assign
//   linear    o = j, c = m,  U = v,   W = b*k, Y = q                   prefix, add
//   alpha     o = r, c = j,  U = b*q, W = w_hat, Y = v                 suffix, assign
//   beta      o = r, c = j,  U = b*q, W = o (.) w_hat, Y = 1           suffix, subtract
// CTA: 32 output features o x 8 slices of c; a thread keeps X[o][c] for its slice in
// registers (MPT = ceil(Dc / 8)); the 8 slice threads of one o are adjacent lanes,
// so the dot over c is 3 xor-shuffles.
struct Src {
  const void* p;  // null: constant 1
  int layout;
  float scale;
};
struct TermArgs {
  Src U, W, W2, Y;  // W2: optional elementwise factor of W (beta's o (.) w_hat)
  float* acc;
  int64_t N, Do, Dc;
  int suffix, mode;  // mode 0 assign, 1 add, 2 subtract
};

constexpr int kTermRows = 32;

template <typename T>
__device__ __forceinline__ void load_rows(float* dst, int ld_dst, const Src& s, const Src* s2, int64_t g, int64_t N,
                                          int64_t Dfull, int64_t c0, int64_t cn, int64_t t0, int rows) {
  // dst[li * ld_dst + c] = s(g, t0 + li, c0 + c) (* s2(...)) * scale, li < rows, c < cn;
  // zero elsewhere up to kTermRows x ld_dst. Index order follows the source layout.
  const int tid = threadIdx.x, nt = blockDim.x;
  const int total = kTermRows * ld_dst;
  const bool fm = s.layout == LA_FEATURE_MAJOR;
  for (int e = tid; e < total; e += nt) {
    const int li = fm ? e % kTermRows : e / ld_dst;
    const int c = fm ? e / kTermRows : e % ld_dst;
    float v = 0.f;
    if (li < rows && c < cn) {
      const int64_t t = t0 + li, cc = c0 + c;
      if (s.p == nullptr) {
        v = s.scale;
      } else {
        const T* base = (const T*)s.p + g * N * Dfull;
        v = ld(base + (fm ? cc * N + t : t * Dfull + cc)) * s.scale;
        if (s2 && s2->p) {
          const T* b2 = (const T*)s2->p + g * N * Dfull;
          v *= ld(b2 + (s2->layout == LA_FEATURE_MAJOR ? cc * N + t : t * Dfull + cc)) * s2->scale;
        }
      }
    }
    dst[li * ld_dst + c] = v;
  }
}

template <typename T, int MPT>
__global__ void __launch_bounds__(256) k_term_sweep(TermArgs a) {
  extern __shared__ float sm[];
  const int Dc8 = 8 * MPT;                       // padded c extent
  float* Ut = sm;                                // [rows][32]
  float* Wt = Ut + kTermRows * 32;               // [rows][Dc8]
  float* Yt = Wt + kTermRows * Dc8;              // [rows][Dc8]
  float* Ot = Yt + kTermRows * Dc8;              // [32 o][rows + 1]
  const int64_t g = blockIdx.y, o0 = (int64_t)blockIdx.x * 32;
  const int ol = threadIdx.x / 8, sl = threadIdx.x % 8;
  float X[MPT];
#pragma unroll
  for (int r = 0; r < MPT; ++r) X[r] = 0.f;
  const int64_t ntiles = (a.N + kTermRows - 1) / kTermRows;
  for (int64_t tt = 0; tt < ntiles; ++tt) {
    const int64_t tile = a.suffix ? ntiles - 1 - tt : tt;
    const int64_t t0 = tile * kTermRows;
    const int rows = (int)lmin(kTermRows, a.N - t0);
    __syncthreads();
    load_rows<T>(Ut, 32, a.U, nullptr, g, a.N, a.Do, o0, lmin(32, a.Do - o0), t0, rows);
    load_rows<T>(Wt, Dc8, a.W, &a.W2, g, a.N, a.Do, 0, a.Dc, t0, rows);  // tensors are (G, N, Do)
    load_rows<T>(Yt, Dc8, a.Y, nullptr, g, a.N, a.Do, 0, a.Dc, t0, rows);
    __syncthreads();
    for (int k = 0; k < rows; ++k) {
      const int li = a.suffix ? rows - 1 - k : k;
      const float u = Ut[li * 32 + ol];
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < MPT; ++r) {
        const int c = sl + 8 * r;
        X[r] += u * Wt[li * Dc8 + c];
        acc += X[r] * Yt[li * Dc8 + c];
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (sl == 0) Ot[ol * (kTermRows + 1) + li] = acc;
    }
    __syncthreads();
    // coalesced along t: acc[g][o][t]
    for (int e = threadIdx.x; e < 32 * kTermRows; e += blockDim.x) {
      const int li = e % kTermRows, oo = e / kTermRows;
      if (li >= rows || o0 + oo >= a.Do) continue;
      float* dst = a.acc + (g * a.Do + o0 + oo) * a.N + t0 + li;
      const float v = Ot[oo * (kTermRows + 1) + li];
      *dst = a.mode == 0 ? v : (a.mode == 1 ? *dst + v : *dst - v);
    }
  }
}

template <typename T>
cudaError_t launch_term(const TermArgs& a, int64_t G, cudaStream_t s) {
  const int mpt = a.Dc <= 32 ? 4 : a.Dc <= 64 ? 8 : a.Dc <= 128 ? 16 : 32;
  const size_t smem = sizeof(float) * (kTermRows * 32 + 2 * kTermRows * 8 * mpt + 32 * (kTermRows + 1));
  const dim3 grid((unsigned)((a.Do + 31) / 32), (unsigned)G);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, s>>>(a);
  };
  switch (mpt) {
    case 4: go(k_term_sweep<T, 4>); break;
    case 8: go(k_term_sweep<T, 8>); break;
    case 16: go(k_term_sweep<T, 16>); break;
    default: go(k_term_sweep<T, 32>); break;
  }
  note_launch(1);
  return cudaGetLastError();
}

cudaError_t dispatch_term(int dtype, const TermArgs& a, int64_t G, cudaStream_t s) {
  if (dtype == LA_F32) return launch_term<float>(a, G, s);
  if (dtype == LA_BF16) return launch_term<__nv_bfloat16>(a, G, s);
  return launch_term<__half>(a, G, s);
}

// ------------------------------------------------------------------ validation
la_status fail(la_error_info* err, la_status code, const char* msg) {
  if (err) {
    err->code = code;
    err->group = err->position = -1;
    std::snprintf(err->message, sizeof(err->message), "%s", msg);
  }
  return code;
}
la_status done(la_error_info* err, cudaError_t e) {
  if (e != cudaSuccess) {
    char buf[200];
    std::snprintf(buf, sizeof(buf), "CUDA error: %s", cudaGetErrorString(e));
    return fail(err, LA_ERR_CUDA, buf);
  }
  if (err) {
    err->code = LA_OK;
    err->group = err->position = -1;
    err->message[0] = 0;
  }
  return LA_OK;
}
bool lay_ok(int l) { return l == LA_FEATURE_MAJOR || l == LA_SEQUENCE_MAJOR; }
la_status base_checks(const la_problem* p, la_error_info* err, const char* empty_msg) {
  if (!p) return fail(err, LA_ERR_INVALID_ARGUMENT, "null problem");
  if (p->groups <= 0 || p->seq_len <= 0 || p->dim <= 0) return fail(err, LA_ERR_INVALID_SHAPE, empty_msg);
  if (p->dtype != LA_F32 && p->dtype != LA_BF16 && p->dtype != LA_F16)
    return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (p->dim > 256) return fail(err, LA_ERR_UNSUPPORTED, "head dimension above 256");
  return LA_OK;
}

}  // namespace
}  // namespace lab

using namespace lab;

extern "C" {

la_status la_normalize_qk(const la_problem* p, const void* q, la_layout lq, const void* k, la_layout lk,
                          void* q_out, void* k_out, void* stream, la_error_info* err) {
  la_status st = base_checks(p, err, "normalize_qk requires non-empty Q and K");
  if (st != LA_OK) return st;
  if (!q || !k || !q_out || !k_out) return fail(err, LA_ERR_INVALID_ARGUMENT, "null tensor");
  if (!lay_ok(lq) || !lay_ok(lk)) return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  const cudaStream_t s = (cudaStream_t)stream;
  const int64_t G = p->groups, N = p->seq_len;
  const int D = (int)p->dim;
  auto one = [&](const void* x, la_layout l, void* y) {
    auto run = [&](auto* tag) {
      using T = std::remove_pointer_t<decltype(tag)>;
      if (l == LA_SEQUENCE_MAJOR)
        k_normalize_seq<T><<<(unsigned)((G * N + 7) / 8), 256, 0, s>>>((const T*)x, (T*)y, G * N, D);
      else
        k_normalize_feat<T><<<dim3((unsigned)((N + 255) / 256), (unsigned)G), 256, 0, s>>>((const T*)x, (T*)y, G, N, D);
    };
    if (p->dtype == LA_F32) run((float*)nullptr);
    else if (p->dtype == LA_BF16) run((__nv_bfloat16*)nullptr);
    else run((__half*)nullptr);
    note_launch(1);
  };
  one(q, lq, q_out);
  one(k, lk, k_out);
  return done(err, cudaGetLastError());
}

static la_status relayout_impl(const la_problem* p, const void* x, la_layout lx, void* y, la_layout ly,
                               const float* rowdiv, void* stream, la_error_info* err) {
  const cudaStream_t s = (cudaStream_t)stream;
  const int64_t G = p->groups, N = p->seq_len, D = p->dim;
  const dim3 grid((unsigned)((N + 31) / 32), (unsigned)((D + 31) / 32), (unsigned)G);
  if (p->dtype == LA_F32)
    k_relayout<float><<<grid, 256, 0, s>>>((const float*)x, lx, (float*)y, ly, N, D, rowdiv);
  else if (p->dtype == LA_BF16)
    k_relayout<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)x, lx, (__nv_bfloat16*)y, ly, N, D, rowdiv);
  else
    k_relayout<__half><<<grid, 256, 0, s>>>((const __half*)x, lx, (__half*)y, ly, N, D, rowdiv);
  note_launch(1);
  return done(err, cudaGetLastError());
}

la_status la_relayout(const la_problem* p, const void* x, la_layout lx, void* y, la_layout ly, void* stream,
                      la_error_info* err) {
  la_status st = base_checks(p, err, "relayout of an empty tensor");
  if (st != LA_OK) return st;
  if (!x || !y) return fail(err, LA_ERR_INVALID_ARGUMENT, "null tensor");
  if (!lay_ok(lx) || !lay_ok(ly)) return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  if (lx == ly && x == y) return done(err, cudaSuccess);  // the reference shares the buffer
  return relayout_impl(p, x, lx, y, ly, nullptr, stream, err);
}

la_status la_make_omega_hat(const la_problem* p, const void* omega, la_layout lw, const float* g, void* out,
                            void* stream, la_error_info* err) {
  la_status st = base_checks(p, err, "make_omega_hat requires a non-empty cotangent");
  if (st != LA_OK) return st;
  if (!g) return fail(err, LA_ERR_MISSING_FORWARD_STATE, "denominator vector length must equal groups*seq_len");
  if (!omega || !out) return fail(err, LA_ERR_INVALID_ARGUMENT, "null tensor");
  if (!lay_ok(lw)) return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  return relayout_impl(p, omega, lw, out, LA_FEATURE_MAJOR, g, stream, err);
}

la_status la_constant_term_pass(const la_problem* p, const void* v, la_layout lv, float* f, void* stream,
                                la_error_info* err) {
  la_status st = base_checks(p, err, "constant_term_pass requires a non-empty V");
  if (st != LA_OK) return st;
  if (!v || !f) return fail(err, LA_ERR_INVALID_ARGUMENT, "null tensor");
  if (!lay_ok(lv)) return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  TermArgs a{{v, lv, (float)p->a}, {nullptr, 0, 1.f}, {nullptr, 0, 1.f}, {nullptr, 0, 1.f},
             f, p->seq_len, p->dim, 1, 0, 0};
  return done(err, dispatch_term(p->dtype, a, p->groups, (cudaStream_t)stream));
}

la_status la_linear_term_pass(const la_problem* p, const void* q, la_layout lq, const void* k, la_layout lk,
                              const void* v, la_layout lv, float* f, void* stream, la_error_info* err) {
  la_status st = base_checks(p, err, "forward requires non-empty Q, K, V");
  if (st != LA_OK) return st;
  if (p->a == 0.0 && p->b == 0.0)
    return fail(err, LA_ERR_INVALID_ARGUMENT, "kernel coefficients (a, b) must not both be zero");
  st = la_validate_plan(&p->plan, p->groups, p->dim, err);
  if (st != LA_OK) return st;
  if (!q || !k || !v || !f) return fail(err, LA_ERR_INVALID_ARGUMENT, "null tensor");
  if (!lay_ok(lq) || !lay_ok(lk) || !lay_ok(lv)) return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  TermArgs a{{v, lv, 1.f}, {k, lk, (float)p->b}, {nullptr, 0, 1.f}, {q, lq, 1.f},
             f, p->seq_len, p->dim, p->dim, 0, 1};
  return done(err, dispatch_term(p->dtype, a, p->groups, (cudaStream_t)stream));
}

la_status la_alpha_term_pass(const la_problem* p, const void* q, la_layout lq, const void* v, la_layout lv,
                             const void* omega_hat, la_layout lw, float* dk, void* stream, la_error_info* err) {
  la_status st = base_checks(p, err, "term passes require non-empty inputs");
  if (st != LA_OK) return st;
  st = la_validate_plan(&p->plan, p->groups, p->dim, err);
  if (st != LA_OK) return st;
  if (!q || !v || !omega_hat || !dk) return fail(err, LA_ERR_INVALID_ARGUMENT, "null tensor");
  if (!lay_ok(lq) || !lay_ok(lv) || !lay_ok(lw)) return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  TermArgs a{{q, lq, (float)p->b}, {omega_hat, lw, 1.f}, {nullptr, 0, 1.f}, {v, lv, 1.f},
             dk, p->seq_len, p->dim, p->dim, 1, 0};
  return done(err, dispatch_term(p->dtype, a, p->groups, (cudaStream_t)stream));
}

la_status la_beta_term_pass(const la_problem* p, const void* q, la_layout lq, const void* o, la_layout lo,
                            const void* omega_hat, la_layout lw, float* dk, void* stream, la_error_info* err) {
  la_status st = base_checks(p, err, "term passes require non-empty inputs");
  if (st != LA_OK) return st;
  st = la_validate_plan(&p->plan, p->groups, p->dim, err);
  if (st != LA_OK) return st;
  if (!q || !o || !omega_hat || !dk) return fail(err, LA_ERR_INVALID_ARGUMENT, "null tensor");
  if (!lay_ok(lq) || !lay_ok(lo) || !lay_ok(lw)) return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  TermArgs a{{q, lq, (float)p->b}, {o, lo, 1.f}, {omega_hat, lw, 1.f}, {nullptr, 0, 1.f},
             dk, p->seq_len, p->dim, p->dim, 1, 2};
  return done(err, dispatch_term(p->dtype, a, p->groups, (cudaStream_t)stream));
}

}  // extern "C"
