// Internal host-side interfaces between the C-ABI layer and the kernel files.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/la_cuda.h"

namespace lab {

// Per-(group, segment) state record, fp32:
//   [X: D*D row-major][vA: D][vB: D][count: 1]
// forward  (SUM_KV): X[m][j] = sum k_m v_j, vA = sum k (z), vB = sum v (sigma)
// backward (SUM_QW): X[m][j] = sum q_m w_hat_j (R), vA = sum s q (u), vB = sum w_hat (c)
#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t state_floats(int64_t d) { return (d * d + 2 * d + 1 + 3) & ~(int64_t)3; }  // 16-byte records

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
  cudaStream_t stream;
};

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
cudaError_t tc_forward(const Launch& L, const Tensors& t, void* out, float* g, Workspace ws);
cudaError_t tc_backward(const Launch& L, const Tensors& t, void* dq, void* dk, void* dv,
                        Workspace ws);

void note_launch(int n = 1);

// Optional per-kernel event timing (la_profile_enable). Construct before a
// launch and destroy after it; records only while profiling is on.
struct ProfScope {
  ProfScope(const char* name, cudaStream_t s);
  ~ProfScope();
  int idx;
  cudaStream_t stream;
};

}  // namespace lab
