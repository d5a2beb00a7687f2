// Internal host-side interfaces between the C-ABI layer and the kernel files.
#pragma once
#include <algorithm>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/la_cuda.h"

namespace lab {

// Measurement overrides (la_set_tuning); every field 0 unless a benchmark set it.
const la_tuning& tuning();

// Per-(group, segment) state record, fp32:
//   [X: D*D row-major][vA: D][vB: D][count: 1]
// forward  (SUM_KV): X[m][j] = sum k_m v_j, vA = sum k (z), vB = sum v (sigma)
// backward (SUM_QW): X[m][j] = sum q_m w_hat_j (R), vA = sum s q (u), vB = sum w_hat (c)
#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t state_floats(int64_t d) { return (d * d + 2 * d + 1 + 3) & ~(int64_t)3; }  // 16-byte records

// Sequence segmentation shared by the tensor-core forward and backward so a
// forward's saved per-segment states line up with the backward's segments.
// Segments are whole multiples of 128 rows. Rule: the most segments that still fit
// the G x P sweep grid in ONE wave of CTAs (one CTA per SM). Measured on B200 (B=4
// H=16 D=128 bf16, profiles/r01_s3_segments.md): more waves of shorter segments lose
// to the per-CTA prologue (record combine, TMEM / barrier setup), the partial last
// wave and the larger aggregate pre-pass; fewer segments leave SMs idle. At the north
// star (G = 64) this gives P = 2: fwd + bwd 3.26 ms against 3.54 ms at P = 9.
inline int choose_segments(int64_t G, int64_t N, int num_sms = 148) {
  const int64_t c128 = N / 128;
  if (c128 <= 1) return 1;
  int64_t P = G >= num_sms ? 1 : num_sms / G;
  if (P > c128) P = c128;
  if (P > 64) P = 64;
  if (P < 1) P = 1;
  while (P > 1 && ((c128 + P - 1) / P) * (P - 1) >= c128) --P;  // no empty trailing segment
  return (int)P;
}

// Aggregate passes split each segment into A equal units (whole 128-row chunks)
// so that the G x (segments aggregated) x A grid fills the SMs; records are kept
// per unit and summed by the consumer's prologue.
inline int agg_split(int64_t G, int64_t seg_rows, int segs_aggregated, int num_sms = 148) {
  if (segs_aggregated <= 0) return 1;
  const int64_t units = G * segs_aggregated, chunks = seg_rows / 128;
  if (const int a = tuning().agg_split) {  // measurement override
    if (a >= 1 && chunks % a == 0) return a;
  }
  int best = 1;
  double best_t = 1e300;
  for (int A = 1; A <= 8; ++A) {
    if (chunks % A) continue;
    // makespan in whole-segment times: waves of A-way split units, plus a small
    // per-CTA overhead that keeps the split from growing without need
    const double t = (double)((units * A + num_sms - 1) / num_sms) / A + 0.02 * A;
    if (t < best_t - 1e-9) {
      best_t = t;
      best = A;
    }
  }
  return best;
}

// Segment carries: the sweeps sum their carry from the aggregate unit records in their
// prologue, unless the longest such chain ((P - 1) A records) exceeds this -- then one seg_scan
// launch (la_sm100.cu) forms every segment's carry.
constexpr int kScanMinRecords = 8;

// The backward aggregate (W_hat^T / s for every row, R records for segments >= 1): its
// segment-0 units skip Q and the MMAs, so units are uneven; the finest split (up to 8
// units per segment, several waves) balances them (0.70 -> 0.64 ms at the north star).
inline int bwd_agg_split(int64_t seg_rows, int P, bool saved) {
  const int64_t chunks = seg_rows / 128;
  if (const int a = tuning().agg_split) {
    if (a >= 1 && chunks % a == 0) return a;
  }
  // with several segments, a sweep CTA sums (P - 1) A unit records for its R carry: keep that
  // within the in-kernel combine's reach (no scan launch; tiny units cost more than they
  // balance: config-3 shard 0.142 -> 0.119 ms at A = 1). Without the forward's saved states
  // the unit boundaries are also the S rebuild's exact reload points, so keep them fine.
  const int amax = (P > 1 && saved) ? std::max(1, kScanMinRecords / (P - 1)) : 8;
  for (int a = std::min(8, amax); a > 1; --a)
    if (chunks % a == 0) return a;
  return 1;
}

// Causal backward as 2-CTA clusters (la_bwd_pair.cu): one pair sweeps a whole group, the
// W_hat pass fused in, one launch. Used with the forward's saved states when the pairs
// fill the GPU in about one wave; otherwise the segmented single-CTA sweep.
inline bool bwd_pair_rule(int64_t G, int num_sms = 148) {
  if (const int t = tuning().bwd_pair) return t > 0;
  (void)G;
  (void)num_sms;
  return false;  // opt-in until it beats the segmented sweep
}


struct Tensors {
  const void* q; int lq;
  const void* k; int lk;
  const void* v; int lv;
  const void* o; int lo;
  const void* w; int lw;
  const float* g;
};

struct Launch {
  int64_t G, N, D;
  la_dtype dtype;
  float a, b;
  int causal;
  int fault;
  int64_t row_offset;        // sequence sharding: global index of row 0
  int64_t n_total;           // non-causal normaliser length (a * N_total)
  const float* carry_prefix; // G * state_floats(D) or null
  const float* carry_suffix; // G * state_floats(D) or null
  float* saved_out;          // forward: per-(group, segment) end states (la_forward_save) or null
  const float* saved_in;     // backward: the same, from the paired forward, or null
  cudaStream_t stream;
};

// Saved-state buffer (la_forward_save -> la_backward_saved): a 16-float header
// {magic, G, N, D, P, seg_rows, ckK, ckC0} then G * P state records (inclusive prefix
// at each segment's last row: S, z, sigma, rows), then G * ckK checkpoint records.
constexpr float kSavedMagic = 1279348566.0f;  // 'LASV'
constexpr int kSavedHeader = 16;

// Prefix-state checkpoints (tensor-core causal path). The backward's reverse sweep
// rebuilds each chunk's exclusive prefix S (and z) by subtracting K^T V from a later
// exact state. The tensor core's fp32 accumulation truncates every step relative to
// the accumulator's magnitude, so the absolute error grows with the number of steps
// times |S| -- and dq_i = b (w_i S_i^T - s_i z_i) with w_i = omega_i / g_i ~ 1/i weighs
// it most at small global rows (measured 9e-3 max-abs / 2.6e-2 relative on dq at the
// north star with 32K-row segments). The forward therefore also saves the exact
// prefix at the global rows C0 * 2^k (k < ckK, inside a segment); the backward
// reloads S and z there. Steps since the last reload then stay proportional to i,
// so the error weighed by 1/g_i stays bounded at every row, for O(G log N D^2) bytes.
constexpr int kCkC0 = 1024;
#ifdef __CUDACC__
__host__ __device__
#endif
inline int ck_count(int64_t n) {  // checkpoint rows C0 * 2^k below n
  int k = 0;
  while (((int64_t)kCkC0 << k) < n) ++k;
  return k;
}
#ifdef __CUDACC__
__host__ __device__
#endif
inline int ck_index(int64_t global_row, int K) {  // k with global_row == C0 * 2^k, or -1
  if (global_row <= 0 || global_row % kCkC0) return -1;
  const int64_t q = global_row / kCkC0;
  if (q & (q - 1)) return -1;
  int k = 0;
  while (((int64_t)1 << k) < q) ++k;
  return k < K ? k : -1;
}

// Workspace carving shared by every path.
struct Workspace {
  unsigned long long* flag;  // degenerate (group<<32|pos), ULLONG_MAX when clean
  float* base;               // remaining fp32 scratch
  size_t floats;
};

// SIMT (CUDA-core) path, any dtype / D <= 256 / layout.
int simt_segments(int64_t G, int64_t N, int fault);
size_t simt_forward_ws_floats(int64_t G, int64_t N, int64_t D, int fault);
size_t simt_backward_ws_floats(int64_t G, int64_t N, int64_t D, int fault);
cudaError_t simt_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws);
cudaError_t simt_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv,
                          Workspace ws);
// Shard totals (sequence sharding) and the all-gather combine step.
cudaError_t simt_forward_shard_state(const Launch& L, const Tensors& t, float* state_out);
cudaError_t simt_backward_shard_state(const Launch& L, const Tensors& t, float* state_out,
                                      Workspace ws);
cudaError_t combine_shard_states(int64_t G, int64_t D, const float* gathered, int nshards,
                                 int rank, int suffix, float* carry_out, cudaStream_t s);

// sm_100a tcgen05 path (bf16/fp16, canonical layouts).
bool tc_forward_supported(const Launch& L, const Tensors& t);
bool tc_backward_supported(const Launch& L, const Tensors& t);
size_t tc_forward_ws_floats(int64_t G, int64_t N, int64_t D);
size_t tc_backward_ws_floats(int64_t G, int64_t N, int64_t D);
size_t tc_saved_floats(int64_t G, int64_t N, int64_t D);
int tc_segments(int64_t G, int64_t N);

// Sequence-shard totals on the tensor core (bf16/fp16, D = 128, canonical layouts);
// unit records in caller scratch of tc_shard_state_scratch_floats floats.
size_t tc_shard_state_scratch_floats(int64_t G, int64_t N);
cudaError_t tc_forward_shard_state(const Launch& L, const Tensors& t, float* out, float* units);
cudaError_t tc_backward_shard_state(const Launch& L, const Tensors& t, float* out, float* units);
// {magic, G, N, D, P, seg} into a saved-state buffer, stream-ordered and graph-capturable.
void write_saved_header(void* dst, double g, double n, double d, double p, double seg, cudaStream_t st,
                        int ck_k = 0);

// fp32 inputs on the tensor core (3xTF32, la_f32tc.cu): any layouts, D <= 128 (D % 4 == 0),
// N a multiple of 64, causal and non-causal, the Fault mutations, no shard carries.
bool f32tc_supported(const Launch& L, const Tensors& t);
size_t f32tc_ws_floats(int64_t G, int64_t N, int64_t D);
cudaError_t f32tc_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws);
cudaError_t f32tc_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws);

// Generic 16-bit tensor-core path (la_g16.cu): any layouts, D <= 256 (D % 8 == 0), the
// Fault mutations, N a multiple of 64, causal and non-causal, no shard carries.
bool g16_supported(const Launch& L, const Tensors& t);
size_t g16_ws_floats(int64_t G, int64_t N, int64_t D);
cudaError_t g16_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws);
cudaError_t g16_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws);
// Fault::CausalPrefixOffByOne: the generic paths' chunk-boundary term (la_g16.cu).
cudaError_t offbyone_fix(const Launch& L, const Tensors& t, void* out, const float* g);

// Non-causal tensor-core path for D = 64, 192, 256 (bf16/fp16, canonical layouts; la_full.cu).
bool full_tc_supported(const Launch& L, const Tensors& t, bool bwd);
size_t full_ws_floats(int64_t G, int64_t N, int64_t D);
cudaError_t full_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws);
cudaError_t full_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv, Workspace ws);
cudaError_t tc_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws);
cudaError_t tc_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv,
                        Workspace ws);
cudaError_t tc_backward_pair(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv);
// Non-causal helpers shared by the forward and backward files.
int tc_kv_units(int64_t G, int64_t N);
cudaError_t tc_sum_units(const float* recs, int64_t G, int U, float* tot, cudaStream_t st);
cudaError_t tc_kv_totals(const Launch& L, const Tensors& t, float* units, float* tot);

void note_launch(int n = 1);
// mode 0: exclusive prefix at each segment start, 1: inclusive prefix at each segment end,
// 2: exclusive suffix after each segment end (k_seg_scan, la_sm100.cu)
cudaError_t seg_scan(const float* recs, int64_t G, int U, int A, int64_t SZ, const float* base, float* out,
                     int64_t ostride, int mode, float* unit_pre, cudaStream_t st, const char* name);

// Optional per-kernel event timing (la_profile_enable). Construct before a
// launch and destroy after it; records only while profiling is on.
struct ProfScope {
  ProfScope(const char* name, cudaStream_t s);
  ~ProfScope();
  int idx;
  cudaStream_t stream;
};

}  // namespace lab
