// C-ABI layer (include/la_cuda.h): argument validation with the reference's
// error taxonomy, path selection, workspace carving, the device-side
// degenerate-denominator report, and the host-buffer entry points.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool (nsys / ncu --nvtx) injects

#include "../../include/la_cuda.h"
#include "internal.h"

#include <string>
#include <vector>

namespace lab {
static la_tuning g_tuning{};
const la_tuning& tuning() { return g_tuning; }

static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;

// Every kernel scope is also an NVTX range (SURVEY §5 "tracing": the reference's
// ws::set_phase names, forward_kernels.hpp:218,238 / backward_kernels.hpp:303-372, map
// to the phase ranges of forward_impl / backward_impl; these are the kernels under them).
ProfScope::ProfScope(const char* name, cudaStream_t s) : idx(-1), stream(s) {
  nvtxRangePushA(name);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return;
  ProfRec r;
  r.name = name;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, s);
  g_prof.push_back(r);
  idx = (int)g_prof.size() - 1;
}
ProfScope::~ProfScope() {
  nvtxRangePop();
  if (idx < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (idx < (int)g_prof.size()) cudaEventRecord(g_prof[idx].b, stream);
}

// Saved-state header {magic, G, N, D, P, seg} written by a tiny kernel rather than a
// pageable host copy, so a forward + backward step can be captured in a CUDA graph.
__global__ void k_saved_header(float* dst, float g, float n, float d, float p, float seg, float ck) {
  if (threadIdx.x == 0) {
    dst[0] = kSavedMagic;
    dst[1] = g;
    dst[2] = n;
    dst[3] = d;
    dst[4] = p;
    dst[5] = seg;
    dst[6] = ck;
    dst[7] = (float)kCkC0;
  }
}
void write_saved_header(void* dst, double g, double n, double d, double p, double seg, cudaStream_t st,
                        int ck_k) {
  k_saved_header<<<1, 32, 0, st>>>((float*)dst, (float)g, (float)n, (float)d, (float)p, (float)seg, (float)ck_k);
}

// Saved-state validation on the device: the backward checks the header the forward's
// kernel wrote against the problem's expected segmentation, with no host read (so a
// forward + backward step stays asynchronous and graph-capturable). A mismatch sets the
// workspace flag to kFlagSavedMismatch, reported as MissingForwardState by the call
// (err != NULL) or by la_query_status; the outputs are then unspecified.
constexpr unsigned long long kFlagSavedMismatch = 0xFFFFFFFFFFFFFFFEull;
__global__ void k_saved_check(const float* hdr, float g, float n, float d, float p, float seg, float ck,
                              unsigned long long* flag) {
  if (threadIdx.x == 0) {
    const bool match = hdr[0] == kSavedMagic && hdr[1] == g && hdr[2] == n && hdr[3] == d && hdr[4] == p &&
                       hdr[5] == seg && hdr[6] == ck;
    if (!match) atomicExch(flag, kFlagSavedMismatch);
  }
}
}  // namespace lab

using namespace lab;

namespace {

constexpr size_t kFlagBytes = 256;
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

la_status fail(la_error_info* err, la_status code, const char* msg, int64_t grp = -1,
               int64_t pos = -1) {
  if (err) {
    err->code = code;
    err->group = grp;
    err->position = pos;
    std::snprintf(err->message, sizeof(err->message), "%s", msg);
  }
  return code;
}

la_status ok(la_error_info* err) {
  if (err) {
    err->code = LA_OK;
    err->group = err->position = -1;
    err->message[0] = 0;
  }
  return LA_OK;
}

la_status cuda_fail(la_error_info* err, cudaError_t e) {
  char buf[200];
  std::snprintf(buf, sizeof(buf), "CUDA error: %s", cudaGetErrorString(e));
  return fail(err, LA_ERR_CUDA, buf);
}

// check_forward_inputs (forward.cpp:13-25) + validate_plan (plan.cpp:49-62).
la_status check_problem(const la_problem* p, la_error_info* err) {
  if (!p) return fail(err, LA_ERR_INVALID_ARGUMENT, "null problem");
  if (p->groups <= 0 || p->seq_len <= 0 || p->dim <= 0)
    return fail(err, LA_ERR_INVALID_SHAPE, "forward requires non-empty Q, K, V");
  if (p->a == 0.0 && p->b == 0.0)
    return fail(err, LA_ERR_INVALID_ARGUMENT, "kernel coefficients (a, b) must not both be zero");
  la_status s = la_validate_plan(&p->plan, p->groups, p->dim, err);
  if (s != LA_OK) return s;
  if (p->dtype != LA_F32 && p->dtype != LA_BF16 && p->dtype != LA_F16)
    return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown dtype");
  if (p->dim > 256) return fail(err, LA_ERR_UNSUPPORTED, "head dimension above 256");
  if (p->fault < LA_FAULT_NONE || p->fault > LA_FAULT_DROP_GRAD_V_CONSTANT_TERM)
    return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown fault");
  return LA_OK;
}

bool layout_ok(int l) { return l == LA_FEATURE_MAJOR || l == LA_SEQUENCE_MAJOR; }

Launch make_launch(const la_problem* p, const la_shard* sh, void* stream) {
  Launch L;
  L.G = p->groups;
  L.N = p->seq_len;
  L.D = p->dim;
  L.dtype = p->dtype;
  L.a = (float)p->a;
  L.b = (float)p->b;
  L.causal = p->causal ? 1 : 0;
  L.fault = p->fault;
  L.row_offset = sh ? sh->row_offset : 0;
  L.n_total = p->seq_len;
  L.carry_prefix = sh ? sh->carry_in : nullptr;
  L.carry_suffix = sh ? sh->carry_suffix : nullptr;
  L.saved_out = nullptr;
  L.saved_in = nullptr;
  L.stream = (cudaStream_t)stream;
  return L;
}

bool use_tc(const la_problem* p, bool supported) {
  if (p->impl == LA_IMPL_SIMT) return false;
  return supported;
}

size_t ws_bytes_for(size_t floats) { return kFlagBytes + floats * sizeof(float); }

Workspace carve(void* ws, size_t bytes) {
  Workspace w;
  w.flag = (unsigned long long*)ws;
  w.base = (float*)((char*)ws + kFlagBytes);
  w.floats = bytes > kFlagBytes ? (bytes - kFlagBytes) / sizeof(float) : 0;
  return w;
}

la_status finish(void* ws, cudaStream_t s, la_error_info* err) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(err, e);
  if (!err) return LA_OK;  // asynchronous mode: la_query_status later
  return la_query_status(ws, s, err);
}

size_t fwd_floats(const la_problem* p) {
  size_t a = simt_forward_ws_floats(p->groups, p->seq_len, p->dim, p->fault);
  size_t b = std::max(tc_forward_ws_floats(p->groups, p->seq_len, p->dim),
                      full_ws_floats(p->groups, p->seq_len, p->dim));
  if (p->dtype == LA_F32) b = std::max(b, f32tc_ws_floats(p->groups, p->seq_len, p->dim));
  else b = std::max(b, g16_ws_floats(p->groups, p->seq_len, p->dim));
  return a > b ? a : b;
}
size_t bwd_floats(const la_problem* p) {
  size_t a = simt_backward_ws_floats(p->groups, p->seq_len, p->dim, p->fault);
  size_t b = std::max(tc_backward_ws_floats(p->groups, p->seq_len, p->dim),
                      full_ws_floats(p->groups, p->seq_len, p->dim));
  if (p->dtype == LA_F32) b = std::max(b, f32tc_ws_floats(p->groups, p->seq_len, p->dim));
  else b = std::max(b, g16_ws_floats(p->groups, p->seq_len, p->dim));
  return a > b ? a : b;
}

// Head dimensions below 128 on the tensor-core path, canonical layouts, no fault:
// zero-pad D to 128 in device scratch (exact: padded key features add nothing to S or
// z, padded value features are dropped on the way out), run the D = 128 kernels, copy
// the D columns back. Measured faster than the generic kernel at D = 32 / 64 (4.4 vs
// 6.6 ms fwd+bwd at B4 H16 N32768). Non-causal D = 64 has its own kernels (la_full.cu);
// faults and other layouts take the generic kernel (la_g16.cu).
bool pad_eligible(const la_problem* p, const la_shard* sh, int lq, int lk, int lv, int lw) {
  return p->impl != LA_IMPL_SIMT && (p->causal || p->dim != 64) && (p->dtype == LA_BF16 || p->dtype == LA_F16) &&
         p->dim < 128 &&
         p->dim % 8 == 0 && p->fault == LA_FAULT_NONE && p->seq_len % 128 == 0 && sh == nullptr &&
         lq == LA_SEQUENCE_MAJOR && lk == LA_SEQUENCE_MAJOR && lv == LA_FEATURE_MAJOR &&
         (lw < 0 || lw == LA_FEATURE_MAJOR) && p->groups * p->seq_len < (1ll << 31);
}
la_problem padded_problem(const la_problem* p) {
  la_problem q = *p;
  q.dim = 128;
  la_default_plan(q.groups, 128, p->plan.workers > 0 ? p->plan.workers : 1, &q.plan);
  return q;
}
// Sequence lengths that are not a multiple of 128 on the tensor-core path: the rows
// are zero-padded to Np = 128 * ceil(N / 128) in device scratch. Exact for both masks:
// padded keys / values add nothing to any state, padded cotangent rows (omega = 0)
// give w_hat = 0, padded rows come after every real row (causal prefixes of real rows
// are unchanged) and the non-causal normaliser keeps a * N (n_total). Padded rows have
// g = a (i + 1) or a N, so a >= 1e-3 keeps them away from the degenerate threshold.
bool padn_eligible(const la_problem* p, const la_shard* sh, int lq, int lk, int lv, int lw) {
  const int64_t np = (p->seq_len + 127) / 128 * 128;
  // D <= 128: tcgen05 (D < 128 through the D padding); non-causal D = 192, 256: la_full.cu;
  // causal D = 192, 256 only when N is not a multiple of the generic path's 64-row chunk
  // (la_g16.cu takes the shape as it is otherwise)
  const bool fast_d = p->dim <= 128 || (!p->causal && (p->dim == 192 || p->dim == 256)) ||
                      (p->dim <= 256 && p->seq_len % 64 != 0);
  return p->impl != LA_IMPL_SIMT && (p->dtype == LA_BF16 || p->dtype == LA_F16) && p->seq_len % 128 != 0 &&
         fast_d && p->dim % 8 == 0 && p->fault == LA_FAULT_NONE && p->a >= 1e-3 && sh == nullptr &&
         lq == LA_SEQUENCE_MAJOR && lk == LA_SEQUENCE_MAJOR && lv == LA_FEATURE_MAJOR &&
         (lw < 0 || lw == LA_FEATURE_MAJOR) && p->groups * np * (p->dim + 8) < (1ll << 31);
}
la_problem n_padded_problem(const la_problem* p) {
  la_problem q = *p;
  q.seq_len = (p->seq_len + 127) / 128 * 128;
  return q;
}
// rows x w elements from a row pitch of sp to dp elements; the tail [w, wd) of every
// destination row is set to `fill` (wd = w copies back without a tail). One pass, 4
// consecutive elements per thread (rows are not 16-byte aligned when N is odd).
template <typename T>
__global__ void k_pitch_copy(T* dst, int64_t dp, const T* src, int64_t sp, int64_t w, int64_t wd, T fill) {
  const int64_t r = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * 2048 + threadIdx.x;  // element c0 + 256 u: warps stay contiguous
  T v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = c0 + 256 * u < w ? src[r * sp + c0 + 256 * u] : fill;  // 8 loads in flight
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (c0 + 256 * u < wd) dst[r * dp + c0 + 256 * u] = v[u];
}
// 16-byte variant: every row start, pitch and w a multiple of 16 bytes.
template <typename T>
__global__ void k_pitch_copy16(uint4* dst, int64_t dp, const uint4* src, int64_t sp, int64_t w, int64_t wd,
                               T fill) {
  const int64_t r = blockIdx.y;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // 16-byte vector index
  if (c >= wd) return;
  uint4 f;
  T* fe = (T*)&f;
#pragma unroll
  for (int u = 0; u < (int)(16 / sizeof(T)); ++u) fe[u] = fill;
  dst[r * dp + c] = c < w ? src[r * sp + c] : f;
}
template <typename T>
void pitch_copy(T* dst, int64_t dp, const T* src, int64_t sp, int64_t w, int64_t wd, int64_t rows, T fill,
                cudaStream_t st) {
  constexpr int64_t V = 16 / sizeof(T);
  if (dp % V == 0 && sp % V == 0 && w % V == 0 && wd % V == 0 && ((uintptr_t)dst | (uintptr_t)src) % 16 == 0) {
    const dim3 grid((unsigned)((wd / V + 255) / 256), (unsigned)rows);
    k_pitch_copy16<T><<<grid, 256, 0, st>>>((uint4*)dst, dp / V, (const uint4*)src, sp / V, w / V, wd / V, fill);
  } else {
    const dim3 grid((unsigned)((wd + 2047) / 2048), (unsigned)rows);
    k_pitch_copy<T><<<grid, 256, 0, st>>>(dst, dp, src, sp, w, wd, fill);
  }
}
using u16 = unsigned short;

// [rows][D] <-> [rows][128] (SequenceMajor) and [G][D][N] <-> [G][128][N] (FeatureMajor),
// 16-byte vectors, zero fill of the padded part on the way in.
__global__ void k_pad_seq(uint4* dst, const uint4* src, int64_t rows, int dv, int to_padded) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // 16-byte vector of the 128-wide row
  if (e >= rows * 16) return;
  const int64_t r = e >> 4;
  const int c = (int)(e & 15);
  if (to_padded) dst[e] = c < dv ? src[r * dv + c] : make_uint4(0, 0, 0, 0);
  else if (c < dv) dst[r * dv + c] = src[e];
}
__global__ void k_pad_feat(uint4* dst, const uint4* src, int64_t G, int D, int64_t nv, int to_padded) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // vector of the [G][128][N] tensor
  if (e >= G * 128 * nv) return;
  const int64_t g = e / (128 * nv), rem = e % (128 * nv);
  const int j = (int)(rem / nv);
  const int64_t i = rem % nv;
  if (to_padded) dst[e] = j < D ? src[(g * D + j) * nv + i] : make_uint4(0, 0, 0, 0);
  else if (j < D) dst[(g * D + j) * nv + i] = src[e];
}
void pad_copy(void* dst, const void* src, const la_problem* p, bool seq_major, bool to_padded, cudaStream_t st) {
  const int64_t G = p->groups, N = p->seq_len;
  const int D = (int)p->dim;
  if (seq_major) {
    const int64_t n = G * N * 16;
    k_pad_seq<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((uint4*)dst, (const uint4*)src, G * N, D / 8,
                                                           to_padded ? 1 : 0);
  } else {
    const int64_t n = G * 128 * (N / 8);
    k_pad_feat<<<(unsigned)((n + 255) / 256), 256, 0, st>>>((uint4*)dst, (const uint4*)src, G, D, N / 8,
                                                            to_padded ? 1 : 0);
  }
  note_launch(1);
}

// Phase range of one public forward / backward call (the reference's ws::set_phase,
// forward_kernels.hpp:218,238, backward_kernels.hpp:303,327,343,372, one level up: the
// fused kernels compute those term phases together).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

la_status forward_impl(const la_problem* p, const la_shard* sh, const void* q, la_layout lq,
                       const void* k, la_layout lk, const void* v, la_layout lv, void* out,
                       float* g, void* ws, size_t ws_bytes, void* stream, la_error_info* err,
                       void* saved = nullptr, size_t saved_bytes = 0, int64_t n_total = 0) {
  NvtxRange phase(p && !p->causal ? "forward.full" : "forward.causal");
  la_status s = check_problem(p, err);
  if (s != LA_OK) return s;
  if (!q || !k || !v || !out || !g)
    return fail(err, LA_ERR_INVALID_SHAPE, "forward requires non-empty Q, K, V and outputs");
  if (!layout_ok(lq) || !layout_ok(lk) || !layout_ok(lv))
    return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  if (!ws || ws_bytes < la_forward_workspace_bytes(p))
    return fail(err, LA_ERR_WORKSPACE, "workspace smaller than la_forward_workspace_bytes");
  if (sh && !p->causal && (sh->carry_in || sh->row_offset))
    return fail(err, LA_ERR_UNSUPPORTED, "sequence sharding is defined for the causal mask");
  if (padn_eligible(p, sh, lq, lk, lv, -1)) {
    const la_problem pn = n_padded_problem(p);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t G = p->groups, N = p->seq_len, Np = pn.seq_len, D = p->dim;
    const size_t T = (size_t)G * Np * D * 2;
    const size_t inner = align256(la_forward_workspace_bytes(&pn));
    char* buf = (char*)ws + inner;  // the padded copies follow the inner workspace
    pitch_copy<u16>((u16*)buf, Np * D, (const u16*)q, N * D, N * D, Np * D, G, 0, st);  // SequenceMajor rows
    pitch_copy<u16>((u16*)(buf + T), Np * D, (const u16*)k, N * D, N * D, Np * D, G, 0, st);
    pitch_copy<u16>((u16*)(buf + 2 * T), Np, (const u16*)v, N, N, Np, G * D, 0, st);   // FeatureMajor rows
    note_launch(3);
    float* gp = (float*)(buf + 4 * T);
    // the saved states are the padded problem's (la_saved_state_bytes sizes them for Np)
    s = forward_impl(&pn, nullptr, buf, LA_SEQUENCE_MAJOR, buf + T, LA_SEQUENCE_MAJOR, buf + 2 * T,
                     LA_FEATURE_MAJOR, buf + 3 * T, gp, ws, inner, stream, nullptr, saved, saved_bytes, N);
    if (s == LA_OK) {
      pitch_copy<u16>((u16*)out, N, (const u16*)(buf + 3 * T), Np, N, N, G * D, 0, st);
      pitch_copy<float>(g, N, gp, Np, N, N, G, 0.f, st);
      note_launch(2);
    }
    if (s != LA_OK) return fail(err, s, "sequence-padded forward failed");
    return finish(ws, st, err);
  }
  if (pad_eligible(p, sh, lq, lk, lv, -1)) {
    const la_problem p2 = padded_problem(p);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t T = (size_t)p->groups * p->seq_len * 128 * 2;
    const size_t inner = align256(la_forward_workspace_bytes(&p2));
    char* buf = (char*)ws + inner;
    pad_copy(buf, q, p, true, true, st);
    pad_copy(buf + T, k, p, true, true, st);
    pad_copy(buf + 2 * T, v, p, false, true, st);
    if (saved) {  // no per-segment states on this path: header only, the backward recomputes
      write_saved_header(saved, (double)p->groups, (double)p->seq_len, (double)p->dim, 0, 0, st);
    }
    s = forward_impl(&p2, nullptr, buf, LA_SEQUENCE_MAJOR, buf + T, LA_SEQUENCE_MAJOR, buf + 2 * T,
                     LA_FEATURE_MAJOR, buf + 3 * T, g, ws, inner, stream, nullptr, nullptr, 0, n_total);
    if (s == LA_OK) pad_copy(out, buf + 3 * T, p, false, false, st);
    if (s != LA_OK) return fail(err, s, "padded forward failed");
    return finish(ws, st, err);
  }
  Launch L = make_launch(p, sh, stream);
  if (n_total > 0) L.n_total = n_total;  // padded rows excluded from the non-causal a * N
  Tensors t{q, lq, k, lk, v, lv, nullptr, 0, nullptr, 0, nullptr};
  Workspace w = carve(ws, ws_bytes);
  if (saved && saved_bytes < la_saved_state_bytes(p))
    return fail(err, LA_ERR_WORKSPACE, "saved-state buffer smaller than la_saved_state_bytes");
  cudaMemsetAsync(w.flag, 0xFF, sizeof(unsigned long long), L.stream);
  cudaError_t e;
  // la_full.cu first: it takes the non-causal shapes it supports (D = 64 / 128 / 192 / 256);
  // the D = 128 canonical kernels take the rest of D = 128
  const bool full = p->impl != LA_IMPL_SIMT && full_tc_supported(L, t, false);
  const bool tc = !full && use_tc(p, tc_forward_supported(L, t));
  const bool gen = !tc && !full && p->impl != LA_IMPL_SIMT && g16_supported(L, t);
  const bool f32 = !tc && !full && p->impl != LA_IMPL_SIMT && f32tc_supported(L, t);
  if (saved) {
    if (tc || full) {  // causal: prefix states per segment; non-causal: the K/V totals
      L.saved_out = (float*)saved;
    } else {  // header only: the backward recomputes its prefix states
      write_saved_header(saved, (double)p->groups, (double)p->seq_len, (double)p->dim, 0, 0, L.stream);
    }
  }
  if (tc)
    e = tc_forward(L, t, out, g, w);
  else if (full)
    e = full_forward(L, t, out, g, w);
  else if (gen)
    e = g16_forward(L, t, out, g, w);
  else if (f32)
    e = f32tc_forward(L, t, out, g, w);
  else if (p->impl == LA_IMPL_TCGEN05)
    return fail(err, LA_ERR_UNSUPPORTED,
                "tcgen05 path needs bf16/fp16 with D <= 256 (D % 8 == 0), or fp32 with D <= 128 (D % 4 == 0), "
                "and N a multiple of 64, without sequence-shard carries");
  else
    e = simt_forward(L, t, out, g, w);
  if (e != cudaSuccess) return cuda_fail(err, e);
  return finish(ws, L.stream, err);
}

la_status backward_impl(const la_problem* p, const la_shard* sh, const void* q, la_layout lq,
                        const void* k, la_layout lk, const void* v, la_layout lv, const void* o,
                        const void* omega, la_layout lw, const float* g, void* dq, void* dk,
                        void* dv, void* ws, size_t ws_bytes, void* stream, la_error_info* err,
                        const void* saved = nullptr, size_t saved_bytes = 0, bool trust_saved = false) {
  NvtxRange phase(p && !p->causal ? "backward.full" : "backward.causal");
  // check_backward_inputs (backward.cpp:13-28)
  if (p && (!o || !q || !k || !v))
    return fail(err, LA_ERR_MISSING_FORWARD_STATE,
                "backward requires the forward artifacts (Q, K, V, O)");
  if (p && !g)
    return fail(err, LA_ERR_MISSING_FORWARD_STATE, "backward requires the retained denominator vector g");
  if (p && !omega) return fail(err, LA_ERR_SHAPE_MISMATCH, "cotangent shape must match the forward output");
  la_status s = check_problem(p, err);
  if (s != LA_OK) return s;
  if (!dq || !dk || !dv) return fail(err, LA_ERR_INVALID_SHAPE, "null gradient buffer");
  if (!layout_ok(lq) || !layout_ok(lk) || !layout_ok(lv) || !layout_ok(lw))
    return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  if (!ws || ws_bytes < la_backward_workspace_bytes(p))
    return fail(err, LA_ERR_WORKSPACE, "workspace smaller than la_backward_workspace_bytes");
  if (sh && !p->causal && (sh->carry_in || sh->carry_suffix || sh->row_offset))
    return fail(err, LA_ERR_UNSUPPORTED, "sequence sharding is defined for the causal mask");
  if (padn_eligible(p, sh, lq, lk, lv, lw)) {
    const la_problem pn = n_padded_problem(p);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t G = p->groups, N = p->seq_len, Np = pn.seq_len, D = p->dim;
    const size_t T = (size_t)G * Np * D * 2;
    const size_t inner = align256(la_backward_workspace_bytes(&pn));
    char* buf = (char*)ws + inner;  // the padded copies follow the inner workspace
    pitch_copy<u16>((u16*)buf, Np * D, (const u16*)q, N * D, N * D, Np * D, G, 0, st);
    pitch_copy<u16>((u16*)(buf + T), Np * D, (const u16*)k, N * D, N * D, Np * D, G, 0, st);
    pitch_copy<u16>((u16*)(buf + 2 * T), Np, (const u16*)v, N, N, Np, G * D, 0, st);
    pitch_copy<u16>((u16*)(buf + 3 * T), Np, (const u16*)o, N, N, Np, G * D, 0, st);
    pitch_copy<u16>((u16*)(buf + 4 * T), Np, (const u16*)omega, N, N, Np, G * D, 0, st);
    float* gp = (float*)(buf + 8 * T);
    pitch_copy<float>(gp, Np, g, N, N, Np, G, 1.f, st);  // padded rows: w_hat = 0 / 1
    note_launch(6);
    la_status s2 = backward_impl(&pn, nullptr, buf, LA_SEQUENCE_MAJOR, buf + T, LA_SEQUENCE_MAJOR, buf + 2 * T,
                                 LA_FEATURE_MAJOR, buf + 3 * T, buf + 4 * T, LA_FEATURE_MAJOR, gp, buf + 5 * T,
                                 buf + 6 * T, buf + 7 * T, ws, inner, stream, nullptr, saved, saved_bytes,
                                 trust_saved);
    if (s2 == LA_OK) {
      pitch_copy<u16>((u16*)dq, N * D, (const u16*)(buf + 5 * T), Np * D, N * D, N * D, G, 0, st);
      pitch_copy<u16>((u16*)dk, N, (const u16*)(buf + 6 * T), Np, N, N, G * D, 0, st);
      pitch_copy<u16>((u16*)dv, N, (const u16*)(buf + 7 * T), Np, N, N, G * D, 0, st);
      note_launch(3);
    }
    if (s2 != LA_OK) return fail(err, s2, "sequence-padded backward failed");
    return finish(ws, st, err);
  }
  if (pad_eligible(p, sh, lq, lk, lv, lw)) {
    const la_problem p2 = padded_problem(p);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t T = (size_t)p->groups * p->seq_len * 128 * 2;
    const size_t inner = align256(la_backward_workspace_bytes(&p2));
    char* buf = (char*)ws + inner;
    pad_copy(buf, q, p, true, true, st);
    pad_copy(buf + T, k, p, true, true, st);
    pad_copy(buf + 2 * T, v, p, false, true, st);
    pad_copy(buf + 3 * T, o, p, false, true, st);
    pad_copy(buf + 4 * T, omega, p, false, true, st);
    la_status s2 = backward_impl(&p2, nullptr, buf, LA_SEQUENCE_MAJOR, buf + T, LA_SEQUENCE_MAJOR, buf + 2 * T,
                                 LA_FEATURE_MAJOR, buf + 3 * T, buf + 4 * T, LA_FEATURE_MAJOR, g, buf + 5 * T,
                                 buf + 6 * T, buf + 7 * T, ws, inner, stream, nullptr);
    if (s2 == LA_OK) {
      pad_copy(dq, buf + 5 * T, p, true, false, st);
      pad_copy(dk, buf + 6 * T, p, false, false, st);
      pad_copy(dv, buf + 7 * T, p, false, false, st);
    }
    if (s2 != LA_OK) return fail(err, s2, "padded backward failed");
    return finish(ws, st, err);
  }
  Launch L = make_launch(p, sh, stream);
  Tensors t{q, lq, k, lk, v, lv, o, LA_FEATURE_MAJOR, omega, lw, g};
  Workspace w = carve(ws, ws_bytes);
  // la_full.cu first: it takes the non-causal shapes it supports (D = 64 / 128 / 192 / 256);
  // the D = 128 canonical kernels take the rest of D = 128
  const bool full = p->impl != LA_IMPL_SIMT && full_tc_supported(L, t, true);
  const bool tc = !full && use_tc(p, tc_backward_supported(L, t));
  const bool gen = !tc && !full && p->impl != LA_IMPL_SIMT && g16_supported(L, t);
  const bool f32 = !tc && !full && p->impl != LA_IMPL_SIMT && f32tc_supported(L, t);
  cudaMemsetAsync(w.flag, 0xFF, sizeof(unsigned long long), L.stream);
  if (saved && (tc || full)) {
    // states from la_forward_save of the same problem: causal -> per-segment prefixes
    // + checkpoints, non-causal -> the K/V totals (header P = -1)
    if (saved_bytes < la_saved_state_bytes(p))
      return fail(err, LA_ERR_WORKSPACE, "saved-state buffer smaller than la_saved_state_bytes");
    L.saved_in = (const float*)saved;
    if (!trust_saved) {  // la_host_step hands over its own forward's buffer unchecked
      const bool ct = p->causal && tc;
      const int P = ct ? tc_segments(p->groups, p->seq_len) : -1;
      const int64_t seg = ct ? ((p->seq_len / 128 + P - 1) / P) * 128 : 0;
      k_saved_check<<<1, 32, 0, L.stream>>>((const float*)saved, (float)p->groups, (float)p->seq_len,
                                            (float)p->dim, (float)P, (float)seg,
                                            (float)(ct ? ck_count(p->seq_len) : 0), w.flag);
      note_launch(1);
    }
  }
  cudaError_t e;
  if (tc)
    e = tc_backward(L, t, dq, dk, dv, w);
  else if (full)
    e = full_backward(L, t, dq, dk, dv, w);
  else if (gen)
    e = g16_backward(L, t, dq, dk, dv, w);
  else if (f32)
    e = f32tc_backward(L, t, dq, dk, dv, w);
  else if (p->impl == LA_IMPL_TCGEN05)
    return fail(err, LA_ERR_UNSUPPORTED,
                "tcgen05 path needs bf16/fp16 with D <= 256 (D % 8 == 0), or fp32 with D <= 128 (D % 4 == 0), "
                "and N a multiple of 64, without sequence-shard carries");
  else
    e = simt_backward(L, t, dq, dk, dv, w);
  if (e != cudaSuccess) return cuda_fail(err, e);
  return finish(ws, L.stream, err);
}

size_t elem_bytes(la_dtype d) { return d == LA_F32 ? 4 : 2; }

// Per-thread device arena for the host-buffer API.
struct Arena {
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;
  ~Arena() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    if (stream) cudaStreamDestroy(stream);
    ptr = nullptr;
    bytes = 0;
    stream = nullptr;
  }
  cudaError_t reserve(size_t want) {
    if (!stream) {
      cudaError_t e = cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
      if (e != cudaSuccess) return e;
    }
    if (want <= bytes) return cudaSuccess;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
};
thread_local Arena t_arena;

// Host-buffer training step (la_host_step): the groups are cut into blocks and
// each block's H2D copy, fwd+bwd, and D2H copy run on their own streams through
// a ring of device slots, so PCIe traffic in both directions overlaps compute.
// Up to this many group blocks per step: more blocks shorten the pipeline's fill
// (first H2D) and drain (last D2H), which are the only unoverlapped copies.
constexpr int kHostBlocks = 16;

struct HostPipe {
  static constexpr int R = 3;
  cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[R] = {}, ev_cmp[R] = {}, ev_out[R] = {};
  void* slots = nullptr;
  size_t slot_bytes = 0;
  unsigned long long* hflags = nullptr;  // pinned: per block {forward flag, backward flag}
  int nflags = 0;
  ~HostPipe() { release(); }
  void release() {
    if (s_out) cudaStreamSynchronize(s_out);
    if (slots) cudaFree(slots);
    if (hflags) cudaFreeHost(hflags);
    for (int i = 0; i < R; ++i) {
      if (ev_in[i]) cudaEventDestroy(ev_in[i]);
      if (ev_cmp[i]) cudaEventDestroy(ev_cmp[i]);
      if (ev_out[i]) cudaEventDestroy(ev_out[i]);
      ev_in[i] = ev_cmp[i] = ev_out[i] = nullptr;
    }
    for (cudaStream_t* st : {&s_in, &s_cmp, &s_out})
      if (*st) {
        cudaStreamDestroy(*st);
        *st = nullptr;
      }
    slots = nullptr;
    hflags = nullptr;
    slot_bytes = 0;
    nflags = 0;
  }
  cudaError_t reserve(size_t per_slot, int blocks) {
    cudaError_t e = cudaSuccess;
    if (!s_in) {
      for (cudaStream_t* st : {&s_in, &s_cmp, &s_out})
        if ((e = cudaStreamCreateWithFlags(st, cudaStreamNonBlocking)) != cudaSuccess) return e;
      for (int i = 0; i < R; ++i)
        if ((e = cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ev_cmp[i], cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming)) != cudaSuccess)
          return e;
    }
    if (per_slot > slot_bytes) {
      if (slots) cudaFree(slots);
      slots = nullptr;
      slot_bytes = 0;
      if ((e = cudaMalloc(&slots, per_slot * R)) != cudaSuccess) return e;
      slot_bytes = per_slot;
    }
    if (2 * blocks > nflags) {
      if (hflags) cudaFreeHost(hflags);
      hflags = nullptr;
      nflags = 0;
      if ((e = cudaMallocHost((void**)&hflags, sizeof(unsigned long long) * 2 * blocks)) != cudaSuccess) return e;
      nflags = 2 * blocks;
    }
    return e;
  }
};
thread_local HostPipe t_pipe;

}  // namespace

extern "C" {

// Build provenance: build.py links a one-line object holding the source tree's git revision
// and the link time, so a log shows which build a process loaded.
extern "C" const char la_build_id_str[];
const char* la_version(void) {
  static char v[160];
  std::snprintf(v, sizeof(v), "la-b200 0.2 (sm_100a) build %s", la_build_id_str);
  return v;
}

const char* la_status_name(la_status s) {
  switch (s) {
    case LA_OK: return "ok";
    case LA_ERR_INVALID_SHAPE: return "InvalidShape";
    case LA_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case LA_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case LA_ERR_INVALID_PLAN: return "InvalidPlan";
    case LA_ERR_MISSING_FORWARD_STATE: return "MissingForwardState";
    case LA_ERR_DEGENERATE_DENOMINATOR: return "DegenerateDenominator";
    case LA_ERR_CUDA: return "CudaError";
    case LA_ERR_UNSUPPORTED: return "Unsupported";
    case LA_ERR_WORKSPACE: return "WorkspaceError";
  }
  return "unknown";
}

uint64_t la_launch_count(void) { return g_launches.load(); }

void la_set_tuning(const la_tuning* t) { g_tuning = t ? *t : la_tuning{}; }
void la_get_tuning(la_tuning* t) {
  if (t) *t = g_tuning;
}

void la_profile_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
}

int32_t la_profile_read(char* json, size_t cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::string out = "[";
  for (size_t i = 0; i < g_prof.size(); ++i) {
    float ms = -1.f;
    cudaEventSynchronize(g_prof[i].b);
    cudaEventElapsedTime(&ms, g_prof[i].a, g_prof[i].b);
    char buf[160];
    std::snprintf(buf, sizeof(buf), "%s{\"name\": \"%s\", \"ms\": %.6f}", i ? ", " : "",
                  g_prof[i].name.c_str(), ms);
    out += buf;
    cudaEventDestroy(g_prof[i].a);
    cudaEventDestroy(g_prof[i].b);
  }
  out += "]";
  const int32_t n = (int32_t)g_prof.size();
  g_prof.clear();
  if (json && cap) {
    std::snprintf(json, cap, "%s", out.c_str());
  }
  return n;
}

size_t la_shard_state_floats(const la_problem* p) {
  return p ? (size_t)(p->groups * state_floats(p->dim)) : 0;
}

size_t la_saved_state_bytes(const la_problem* p) {
  if (!p || p->groups <= 0 || p->seq_len <= 0 || p->dim <= 0) return kSavedHeader * sizeof(float);
  if (padn_eligible(p, nullptr, LA_SEQUENCE_MAJOR, LA_SEQUENCE_MAJOR, LA_FEATURE_MAJOR, LA_FEATURE_MAJOR)) {
    const la_problem pn = n_padded_problem(p);  // the padded problem's states
    return tc_saved_floats(pn.groups, pn.seq_len, pn.dim) * sizeof(float);
  }
  return tc_saved_floats(p->groups, p->seq_len, p->dim) * sizeof(float);
}

la_status la_forward_save(const la_problem* p, const void* q, la_layout lq, const void* k,
                          la_layout lk, const void* v, la_layout lv, void* out, float* g,
                          void* saved, size_t saved_bytes, void* workspace, size_t ws_bytes,
                          void* stream, la_error_info* err) {
  if (!saved) return fail(err, LA_ERR_INVALID_ARGUMENT, "null saved-state buffer");
  return forward_impl(p, nullptr, q, lq, k, lk, v, lv, out, g, workspace, ws_bytes, stream, err, saved,
                      saved_bytes);
}

la_status la_backward_saved(const la_problem* p, const void* q, la_layout lq, const void* k,
                            la_layout lk, const void* v, la_layout lv, const void* o,
                            const void* omega, la_layout lw, const float* g, const void* saved,
                            size_t saved_bytes, void* dq, void* dk, void* dv, void* workspace,
                            size_t ws_bytes, void* stream, la_error_info* err) {
  return backward_impl(p, nullptr, q, lq, k, lk, v, lv, o, omega, lw, g, dq, dk, dv, workspace, ws_bytes,
                       stream, err, saved, saved_bytes);
}

// The padded paths run the padded problem in the head of the workspace and keep
// their zero-padded copies of the inputs / outputs in its tail: the caller's
// workspace is the only device memory a call uses (no allocation per call).
size_t la_forward_workspace_bytes(const la_problem* p) {
  if (!p || p->groups <= 0 || p->seq_len <= 0 || p->dim <= 0) return kFlagBytes;
  size_t bytes = ws_bytes_for(fwd_floats(p));
  if (padn_eligible(p, nullptr, LA_SEQUENCE_MAJOR, LA_SEQUENCE_MAJOR, LA_FEATURE_MAJOR, -1)) {
    const la_problem pn = n_padded_problem(p);
    const size_t T = (size_t)p->groups * pn.seq_len * p->dim * 2;
    bytes = std::max(bytes, align256(la_forward_workspace_bytes(&pn)) + 4 * T + (size_t)p->groups * pn.seq_len * 4);
  } else if (pad_eligible(p, nullptr, LA_SEQUENCE_MAJOR, LA_SEQUENCE_MAJOR, LA_FEATURE_MAJOR, -1)) {
    const la_problem p2 = padded_problem(p);
    const size_t T = (size_t)p->groups * p->seq_len * 128 * 2;
    bytes = std::max(bytes, align256(la_forward_workspace_bytes(&p2)) + 4 * T);
  }
  return bytes;
}

size_t la_backward_workspace_bytes(const la_problem* p) {
  if (!p || p->groups <= 0 || p->seq_len <= 0 || p->dim <= 0) return kFlagBytes;
  size_t bytes = ws_bytes_for(bwd_floats(p));
  if (padn_eligible(p, nullptr, LA_SEQUENCE_MAJOR, LA_SEQUENCE_MAJOR, LA_FEATURE_MAJOR, LA_FEATURE_MAJOR)) {
    const la_problem pn = n_padded_problem(p);
    const size_t T = (size_t)p->groups * pn.seq_len * p->dim * 2;
    bytes = std::max(bytes, align256(la_backward_workspace_bytes(&pn)) + 8 * T + (size_t)p->groups * pn.seq_len * 4);
  } else if (pad_eligible(p, nullptr, LA_SEQUENCE_MAJOR, LA_SEQUENCE_MAJOR, LA_FEATURE_MAJOR, LA_FEATURE_MAJOR)) {
    const la_problem p2 = padded_problem(p);
    const size_t T = (size_t)p->groups * p->seq_len * 128 * 2;
    bytes = std::max(bytes, align256(la_backward_workspace_bytes(&p2)) + 8 * T);
  }
  return bytes;
}

// validate_plan (plan.cpp:49-62), same order of checks and messages.
la_status la_validate_plan(const la_block_plan* plan, int64_t groups, int64_t dim,
                           la_error_info* err) {
  if (!plan) return fail(err, LA_ERR_INVALID_PLAN, "null plan");
  if (plan->groups != groups)
    return fail(err, LA_ERR_INVALID_PLAN, "plan group count does not match the tensors");
  if (plan->lanes != dim)
    return fail(err, LA_ERR_INVALID_PLAN, "plan lane count does not match the head dimension");
  if (plan->reduction_blocks < 1 || plan->lanes % plan->reduction_blocks != 0)
    return fail(err, LA_ERR_INVALID_PLAN,
                "reduction block count must be >= 1 and divide the head dimension");
  if (plan->workers < 1) return fail(err, LA_ERR_INVALID_PLAN, "worker count must be >= 1");
  return ok(err);
}

// default_plan (plan.cpp:24-47): L = largest divisor of D not above D/32.
la_status la_default_plan(int64_t groups, int64_t dim, int32_t workers, la_block_plan* out) {
  if (groups <= 0 || dim <= 0 || !out) return LA_ERR_INVALID_SHAPE;
  int64_t target = dim / 32;
  if (target < 1) target = 1;
  int64_t l = 1;
  for (int64_t c = target; c >= 1; --c)
    if (dim % c == 0) {
      l = c;
      break;
    }
  out->groups = groups;
  out->reduction_blocks = l;
  out->lanes = dim;
  out->workers = workers > 0 ? workers : 1;
  out->deterministic = 1;
  return LA_OK;
}

la_status la_query_status(const void* workspace, void* stream, la_error_info* err) {
  unsigned long long flag = ULLONG_MAX;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(&flag, workspace, sizeof(flag), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(err, e);
  if (flag == kFlagSavedMismatch)
    return fail(err, LA_ERR_MISSING_FORWARD_STATE,
                "saved forward state does not come from la_forward_save of this problem");
  if (flag != ULLONG_MAX) {
    const int64_t grp = (int64_t)(flag >> 32), pos = (int64_t)(flag & 0xFFFFFFFFull);
    char msg[160];
    std::snprintf(msg, sizeof(msg), "degenerate attention denominator at group %lld, position %lld",
                  (long long)grp, (long long)pos);
    return fail(err, LA_ERR_DEGENERATE_DENOMINATOR, msg, grp, pos);
  }
  return ok(err);
}

la_status la_forward(const la_problem* p, const void* q, la_layout lq, const void* k, la_layout lk,
                     const void* v, la_layout lv, void* out, float* g, void* workspace,
                     size_t ws_bytes, void* stream, la_error_info* err) {
  return forward_impl(p, nullptr, q, lq, k, lk, v, lv, out, g, workspace, ws_bytes, stream, err);
}

la_status la_backward(const la_problem* p, const void* q, la_layout lq, const void* k,
                      la_layout lk, const void* v, la_layout lv, const void* o, const void* omega,
                      la_layout lw, const float* g, void* dq, void* dk, void* dv, void* workspace,
                      size_t ws_bytes, void* stream, la_error_info* err) {
  return backward_impl(p, nullptr, q, lq, k, lk, v, lv, o, omega, lw, g, dq, dk, dv, workspace,
                       ws_bytes, stream, err);
}

la_status la_forward_sharded(const la_problem* p, const la_shard* shard, const void* q,
                             la_layout lq, const void* k, la_layout lk, const void* v,
                             la_layout lv, void* out, float* g, void* workspace, size_t ws_bytes,
                             void* stream, la_error_info* err) {
  return forward_impl(p, shard, q, lq, k, lk, v, lv, out, g, workspace, ws_bytes, stream, err);
}

la_status la_forward_sharded_save(const la_problem* p, const la_shard* shard, const void* q, la_layout lq,
                                  const void* k, la_layout lk, const void* v, la_layout lv, void* out, float* g,
                                  void* saved, size_t saved_bytes, void* workspace, size_t ws_bytes, void* stream,
                                  la_error_info* err) {
  if (!saved) return fail(err, LA_ERR_INVALID_ARGUMENT, "null saved-state buffer");
  return forward_impl(p, shard, q, lq, k, lk, v, lv, out, g, workspace, ws_bytes, stream, err, saved, saved_bytes);
}

la_status la_backward_sharded_saved(const la_problem* p, const la_shard* shard, const void* q, la_layout lq,
                                    const void* k, la_layout lk, const void* v, la_layout lv, const void* o,
                                    const void* omega, la_layout lw, const float* g, const void* saved,
                                    size_t saved_bytes, void* dq, void* dk, void* dv, void* workspace,
                                    size_t ws_bytes, void* stream, la_error_info* err) {
  return backward_impl(p, shard, q, lq, k, lk, v, lv, o, omega, lw, g, dq, dk, dv, workspace, ws_bytes, stream,
                       err, saved, saved_bytes);
}

la_status la_backward_sharded(const la_problem* p, const la_shard* shard, const void* q,
                              la_layout lq, const void* k, la_layout lk, const void* v,
                              la_layout lv, const void* o, const void* omega, la_layout lw,
                              const float* g, void* dq, void* dk, void* dv, void* workspace,
                              size_t ws_bytes, void* stream, la_error_info* err) {
  return backward_impl(p, shard, q, lq, k, lk, v, lv, o, omega, lw, g, dq, dk, dv, workspace,
                       ws_bytes, stream, err);
}

// Shard totals on the tensor core when the tcgen05 kernels take the shape.
static bool shard_state_tc(const la_problem* p, bool canonical) {
  return p->impl != LA_IMPL_SIMT && (p->dtype == LA_BF16 || p->dtype == LA_F16) && p->dim == 128 &&
         p->seq_len % 128 == 0 && p->fault == LA_FAULT_NONE && canonical && p->groups * p->seq_len < (1ll << 31);
}

size_t la_shard_state_workspace_bytes(const la_problem* p) {
  if (!p || p->groups <= 0 || p->seq_len <= 0 || p->dim <= 0) return 256;
  size_t f = (size_t)(p->groups * p->seq_len);  // CUDA-core backward: s_i per row
  if (shard_state_tc(p, true)) f = std::max(f, tc_shard_state_scratch_floats(p->groups, p->seq_len));
  return align256(f * sizeof(float));
}

la_status la_forward_shard_state(const la_problem* p, const void* k, la_layout lk, const void* v,
                                 la_layout lv, float* state_out, void* workspace, size_t ws_bytes,
                                 void* stream) {
  la_status s = check_problem(p, nullptr);
  if (s != LA_OK) return s;
  if (!k || !v || !state_out) return LA_ERR_INVALID_SHAPE;
  if (!workspace || ws_bytes < la_shard_state_workspace_bytes(p)) return LA_ERR_WORKSPACE;
  Launch L = make_launch(p, nullptr, stream);
  Tensors t{nullptr, 0, k, lk, v, lv, nullptr, 0, nullptr, 0, nullptr};
  if (shard_state_tc(p, lk == LA_SEQUENCE_MAJOR && lv == LA_FEATURE_MAJOR))
    return tc_forward_shard_state(L, t, state_out, (float*)workspace) == cudaSuccess ? LA_OK : LA_ERR_CUDA;
  return simt_forward_shard_state(L, t, state_out) == cudaSuccess ? LA_OK : LA_ERR_CUDA;
}

la_status la_backward_shard_state(const la_problem* p, const void* q, la_layout lq,
                                  const void* o, const void* omega, la_layout lw, const float* g,
                                  float* state_out, void* workspace, size_t ws_bytes, void* stream) {
  la_status s = check_problem(p, nullptr);
  if (s != LA_OK) return s;
  if (!q || !o || !omega || !g || !state_out) return LA_ERR_MISSING_FORWARD_STATE;
  if (!workspace || ws_bytes < la_shard_state_workspace_bytes(p)) return LA_ERR_WORKSPACE;
  Launch L = make_launch(p, nullptr, stream);
  Tensors t{q, lq, nullptr, 0, nullptr, 0, o, LA_FEATURE_MAJOR, omega, lw, g};
  if (shard_state_tc(p, lq == LA_SEQUENCE_MAJOR && lw == LA_FEATURE_MAJOR))
    return tc_backward_shard_state(L, t, state_out, (float*)workspace) == cudaSuccess ? LA_OK : LA_ERR_CUDA;
  Workspace w{nullptr, (float*)workspace, (size_t)(p->groups * p->seq_len)};  // s_i scratch
  return simt_backward_shard_state(L, t, state_out, w) == cudaSuccess ? LA_OK : LA_ERR_CUDA;
}

la_status la_combine_shard_states(const la_problem* p, const float* gathered, int32_t nshards,
                                  int32_t rank, int32_t suffix, float* carry_out, void* stream) {
  if (!p || !gathered || !carry_out || nshards < 1 || rank < 0 || rank >= nshards)
    return LA_ERR_INVALID_ARGUMENT;
  return combine_shard_states(p->groups, p->dim, gathered, nshards, rank, suffix, carry_out,
                              (cudaStream_t)stream) == cudaSuccess
             ? LA_OK
             : LA_ERR_CUDA;
}

la_status la_host_forward(const la_problem* p, const void* q, la_layout lq, const void* k,
                          la_layout lk, const void* v, la_layout lv, void* out, float* g,
                          la_error_info* err) {
  la_status s = check_problem(p, err);
  if (s != LA_OK) return s;
  if (!q || !k || !v || !out || !g) return fail(err, LA_ERR_INVALID_SHAPE, "null host buffer");
  const size_t tb = (size_t)(p->groups * p->seq_len * p->dim) * elem_bytes(p->dtype);
  const size_t gb = sizeof(float) * (size_t)(p->groups * p->seq_len);
  const size_t wb = la_forward_workspace_bytes(p);
  const size_t need = 4 * align256(tb) + align256(gb) + align256(wb);
  cudaError_t e = t_arena.reserve(need);
  if (e != cudaSuccess) return cuda_fail(err, e);
  char* base = (char*)t_arena.ptr;
  void* dq_ = base;
  void* dk_ = base + align256(tb);
  void* dv_ = base + 2 * align256(tb);
  void* dout = base + 3 * align256(tb);
  float* dg = (float*)(base + 4 * align256(tb));
  void* dws = base + 4 * align256(tb) + align256(gb);
  cudaStream_t st = t_arena.stream;
  cudaMemcpyAsync(dq_, q, tb, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dk_, k, tb, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dv_, v, tb, cudaMemcpyHostToDevice, st);
  s = la_forward(p, dq_, lq, dk_, lk, dv_, lv, dout, dg, dws, wb, st, nullptr);
  if (s != LA_OK) return fail(err, s, "device forward failed");
  cudaMemcpyAsync(out, dout, tb, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(g, dg, gb, cudaMemcpyDeviceToHost, st);
  return la_query_status(dws, st, err);
}

la_status la_host_backward(const la_problem* p, const void* q, la_layout lq, const void* k,
                           la_layout lk, const void* v, la_layout lv, const void* o,
                           const void* omega, la_layout lw, const float* g, void* dq, void* dk,
                           void* dv, la_error_info* err) {
  if (p && (!o || !g))
    return fail(err, LA_ERR_MISSING_FORWARD_STATE, "backward requires the forward artifacts");
  la_status s = check_problem(p, err);
  if (s != LA_OK) return s;
  if (!q || !k || !v || !omega || !dq || !dk || !dv)
    return fail(err, LA_ERR_INVALID_SHAPE, "null host buffer");
  const size_t tb = (size_t)(p->groups * p->seq_len * p->dim) * elem_bytes(p->dtype);
  const size_t gb = sizeof(float) * (size_t)(p->groups * p->seq_len);
  const size_t wb = la_backward_workspace_bytes(p);
  const size_t need = 8 * align256(tb) + align256(gb) + align256(wb);
  cudaError_t e = t_arena.reserve(need);
  if (e != cudaSuccess) return cuda_fail(err, e);
  char* base = (char*)t_arena.ptr;
  void* b[8];
  for (int i = 0; i < 8; ++i) b[i] = base + i * align256(tb);
  float* dg = (float*)(base + 8 * align256(tb));
  void* dws = base + 8 * align256(tb) + align256(gb);
  cudaStream_t st = t_arena.stream;
  cudaMemcpyAsync(b[0], q, tb, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b[1], k, tb, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b[2], v, tb, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b[3], o, tb, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(b[4], omega, tb, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dg, g, gb, cudaMemcpyHostToDevice, st);
  s = la_backward(p, b[0], lq, b[1], lk, b[2], lv, b[3], b[4], lw, dg, b[5], b[6], b[7], dws, wb,
                  st, nullptr);
  if (s != LA_OK) return fail(err, s, "device backward failed");
  cudaMemcpyAsync(dq, b[5], tb, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(dk, b[6], tb, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(dv, b[7], tb, cudaMemcpyDeviceToHost, st);
  return la_query_status(dws, st, err);
}

void la_host_release(void) {
  t_arena.release();
  t_pipe.release();
}

la_status la_host_step(const la_problem* p, const void* q, la_layout lq, const void* k,
                       la_layout lk, const void* v, la_layout lv, const void* omega, la_layout lw,
                       void* out, float* g, void* dq, void* dk, void* dv, la_error_info* err) {
  la_status s = check_problem(p, err);
  if (s != LA_OK) return s;
  if (!q || !k || !v || !omega || !out || !g || !dq || !dk || !dv)
    return fail(err, LA_ERR_INVALID_SHAPE, "null host buffer");
  if (!layout_ok(lq) || !layout_ok(lk) || !layout_ok(lv) || !layout_ok(lw))
    return fail(err, LA_ERR_INVALID_ARGUMENT, "unknown layout");
  const int64_t G = p->groups, N = p->seq_len, D = p->dim;
  const int64_t hb = tuning().host_blocks > 0 ? tuning().host_blocks : kHostBlocks;
  const int64_t Gb = (G + hb - 1) / hb;  // blocks of whole groups
  const int nb = (int)((G + Gb - 1) / Gb);
  la_problem pb = *p;
  const size_t eb = elem_bytes(p->dtype);
  const size_t tb = align256((size_t)(Gb * N * D) * eb), gbb = align256(sizeof(float) * (size_t)(Gb * N));
  // The ragged last block has fewer groups, hence possibly more segments per group
  // (choose_segments), so its saved states / workspaces can exceed the full block's:
  // size every slot for the larger of the two block shapes.
  size_t sb = 0, wf = 0, wbk = 0;
  for (const int64_t gs : {Gb, G - (int64_t)(nb - 1) * Gb}) {
    pb.groups = gs;
    pb.plan.groups = gs;
    sb = std::max(sb, align256(la_saved_state_bytes(&pb)));
    wf = std::max(wf, align256(la_forward_workspace_bytes(&pb)));
    wbk = std::max(wbk, align256(la_backward_workspace_bytes(&pb)));
  }
  const size_t per_slot = 8 * tb + gbb + sb + wf + wbk;
  cudaError_t e = t_pipe.reserve(per_slot, nb);
  if (e != cudaSuccess) return cuda_fail(err, e);
  HostPipe& hp = t_pipe;
  for (int bi = 0; bi < nb; ++bi) {
    const int slot = bi % HostPipe::R;
    const int64_t g0 = bi * Gb, gn = (g0 + Gb <= G) ? Gb : G - g0;
    pb.groups = gn;
    pb.plan.groups = gn;
    const size_t tbytes = (size_t)(gn * N * D) * eb, toff = (size_t)(g0 * N * D) * eb;
    const size_t gbytes = sizeof(float) * (size_t)(gn * N), goff = (size_t)(g0 * N);
    char* base = (char*)hp.slots + slot * hp.slot_bytes;
    char* b[8];
    for (int i = 0; i < 8; ++i) b[i] = base + i * tb;
    float* dg = (float*)(base + 8 * tb);
    char* dsaved = base + 8 * tb + gbb;
    char* dwf = dsaved + sb;
    char* dwb = dwf + wf;
    // copy-in
    if (bi >= HostPipe::R) cudaStreamWaitEvent(hp.s_in, hp.ev_out[slot], 0);
    cudaMemcpyAsync(b[0], (const char*)q + toff, tbytes, cudaMemcpyHostToDevice, hp.s_in);
    cudaMemcpyAsync(b[1], (const char*)k + toff, tbytes, cudaMemcpyHostToDevice, hp.s_in);
    cudaMemcpyAsync(b[2], (const char*)v + toff, tbytes, cudaMemcpyHostToDevice, hp.s_in);
    cudaMemcpyAsync(b[3], (const char*)omega + toff, tbytes, cudaMemcpyHostToDevice, hp.s_in);
    cudaEventRecord(hp.ev_in[slot], hp.s_in);
    // forward (saving its segment states) then backward on the block
    cudaStreamWaitEvent(hp.s_cmp, hp.ev_in[slot], 0);
    s = forward_impl(&pb, nullptr, b[0], lq, b[1], lk, b[2], lv, b[4], dg, dwf, wf, hp.s_cmp, nullptr,
                     dsaved, sb);
    if (s != LA_OK) return fail(err, s, "device forward failed");
    s = backward_impl(&pb, nullptr, b[0], lq, b[1], lk, b[2], lv, b[4], b[3], lw, dg, b[5], b[6], b[7], dwb,
                      wbk, hp.s_cmp, nullptr, dsaved, sb, true);
    if (s != LA_OK) return fail(err, s, "device backward failed");
    cudaEventRecord(hp.ev_cmp[slot], hp.s_cmp);
    // copy-out
    cudaStreamWaitEvent(hp.s_out, hp.ev_cmp[slot], 0);
    cudaMemcpyAsync((char*)out + toff, b[4], tbytes, cudaMemcpyDeviceToHost, hp.s_out);
    cudaMemcpyAsync(g + goff, dg, gbytes, cudaMemcpyDeviceToHost, hp.s_out);
    cudaMemcpyAsync((char*)dq + toff, b[5], tbytes, cudaMemcpyDeviceToHost, hp.s_out);
    cudaMemcpyAsync((char*)dk + toff, b[6], tbytes, cudaMemcpyDeviceToHost, hp.s_out);
    cudaMemcpyAsync((char*)dv + toff, b[7], tbytes, cudaMemcpyDeviceToHost, hp.s_out);
    cudaMemcpyAsync(&hp.hflags[2 * bi], dwf, sizeof(unsigned long long), cudaMemcpyDeviceToHost, hp.s_out);
    cudaMemcpyAsync(&hp.hflags[2 * bi + 1], dwb, sizeof(unsigned long long), cudaMemcpyDeviceToHost, hp.s_out);
    cudaEventRecord(hp.ev_out[slot], hp.s_out);
  }
  e = cudaStreamSynchronize(hp.s_out);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(err, e);
  for (int bi = 0; bi < nb; ++bi) {
    const unsigned long long f = hp.hflags[2 * bi];
    if (f != ULLONG_MAX) {
      const int64_t grp = (int64_t)(f >> 32) + bi * Gb, pos = (int64_t)(f & 0xFFFFFFFFull);
      char msg[160];
      std::snprintf(msg, sizeof(msg), "degenerate attention denominator at group %lld, position %lld",
                    (long long)grp, (long long)pos);
      return fail(err, LA_ERR_DEGENERATE_DENOMINATOR, msg, grp, pos);
    }
  }
  return ok(err);
}

}  // extern "C"
