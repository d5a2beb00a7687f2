/*
 * la_cuda.h — C-ABI of the B200 (sm_100a) linear-attention library.
 *
 * Drop-in for the reference library's forward/backward path
 * (/root/reference/proj/include/la/forward.hpp, backward.hpp): same entry
 * points, same (G = B*H, N, D) tensors and FeatureMajor/SequenceMajor layouts,
 * same coefficients f(x) = a + b*x, same BlockPlan validation, same error
 * taxonomy (error.hpp:10-75) as status codes. Plain pointers and sizes only.
 *
 * Entry point                      replaces (reference file:line)
 * -------------------------------  ---------------------------------------------
 * la_forward(causal=1)             la::forward_causal   src/forward.cpp:133-137
 * la_forward(causal=0)             la::forward_full     src/forward.cpp:139-142
 * la_backward(causal=1)            la::backward_causal  src/backward.cpp:93-96
 * la_backward(causal=0)            la::backward_full    src/backward.cpp:98-101
 * la_host_forward / _backward      the same, over host buffers (copies in/out)
 * la_host_step                     forward then backward over host buffers, pipelined
 * la_forward_shard_state           (new) per-shard (S,z,sigma,count) totals for
 * la_backward_shard_state          (new) sequence sharding, exchanged by the
 *                                  caller over NCCL, fed back as carry-in/out
 * la_sharded_forward / _backward   (new) multi-GPU: batch x head or sequence shards,
 *                                  the state exchange over NCCL inside the call
 * la_validate_plan                 la::validate_plan    src/plan.cpp:49-62
 * la_default_plan                  la::default_plan     src/plan.cpp:24-47
 *
 * Device buffers are caller-owned. Calls are stream-ordered; argument errors
 * return synchronously. The degenerate-denominator check (forward_kernels.hpp:53)
 * runs on the device: when `err` is non-NULL the call synchronises its stream and
 * reports the lexicographically first (group, position), like the reference's
 * first-item rethrow (pool.hpp:36-42); with err == NULL it stays asynchronous and
 * la_query_status() reads the flag later.
 */
#ifndef LA_CUDA_H
#define LA_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LA_OK = 0,
  LA_ERR_INVALID_SHAPE = 1,          /* la::InvalidShape */
  LA_ERR_SHAPE_MISMATCH = 2,         /* la::ShapeMismatch */
  LA_ERR_INVALID_ARGUMENT = 3,       /* la::InvalidArgument */
  LA_ERR_INVALID_PLAN = 4,           /* la::InvalidPlan */
  LA_ERR_MISSING_FORWARD_STATE = 5,  /* la::MissingForwardState */
  LA_ERR_DEGENERATE_DENOMINATOR = 6, /* la::DegenerateDenominator(group, position) */
  LA_ERR_CUDA = 7,                   /* CUDA runtime failure */
  LA_ERR_UNSUPPORTED = 8,            /* dtype/shape the device path does not provide */
  LA_ERR_WORKSPACE = 9               /* workspace too small or misaligned */
} la_status;

typedef enum { LA_FEATURE_MAJOR = 0, LA_SEQUENCE_MAJOR = 1 } la_layout; /* tensor.hpp:15 */
typedef enum { LA_F32 = 0, LA_BF16 = 1, LA_F16 = 2 } la_dtype;

typedef enum { /* fault.hpp:7-15 */
  LA_FAULT_NONE = 0,
  LA_FAULT_FLIP_BETA_K_SIGN = 1,
  LA_FAULT_CAUSAL_PREFIX_OFF_BY_ONE = 2,
  LA_FAULT_DROP_GRAD_V_CONSTANT_TERM = 3
} la_fault;

typedef enum { /* device path selection; AUTO picks tcgen05 when the shape allows */
  LA_IMPL_AUTO = 0,
  LA_IMPL_SIMT = 1,   /* CUDA-core fp32 path: every dtype/D, exact sweep order */
  LA_IMPL_TCGEN05 = 2 /* sm_100a tensor-core chunked path (bf16/fp16; fp32 as 3xTF32) */
} la_impl;

typedef struct { /* la::BlockPlan, plan.hpp:15-21 */
  int64_t groups;
  int64_t reduction_blocks; /* L; must divide lanes. Advisory on the GPU. */
  int64_t lanes;            /* must equal D */
  int32_t workers;          /* must be >= 1. Advisory on the GPU. */
  int32_t deterministic;
} la_block_plan;

typedef struct {
  int64_t groups; /* G = batch * heads */
  int64_t seq_len;
  int64_t dim;
  la_dtype dtype;
  double a, b; /* la::LinearKernelCoeffs, tensor.hpp:30-35 */
  int32_t causal;
  la_fault fault;
  la_impl impl;
  la_block_plan plan;
} la_problem;

typedef struct {
  la_status code;
  int64_t group;    /* DegenerateDenominator::group() */
  int64_t position; /* DegenerateDenominator::position() */
  char message[256];
} la_error_info;

/* Per-shard carry for sequence sharding (row range [row_offset, row_offset + N)
 * of a longer sequence). Each pointer is a device array of G * (D*D + 2*D + 1)
 * fp32 values in the layout documented in DESIGN.md; NULL means "no carry". */
typedef struct {
  int64_t row_offset;      /* global index of this shard's first row */
  const float* carry_in;   /* forward: exclusive prefix (S, z, sigma, count) */
  const float* carry_suffix; /* backward: exclusive suffix (R, u, c) */
} la_shard;

/* Measurement overrides of the built-in schedule rules, for benchmark sweeps only
 * (0 = the built-in rule; results never depend on them beyond fp32 summation order).
 * Process-wide; set between calls, not while a call is in flight. */
typedef struct {
  int32_t segments;      /* causal tensor-core segments per group (choose_segments) */
  int32_t agg_split;     /* aggregate-pass units per segment (agg_split / bwd_agg_split) */
  int32_t full_ctas_fwd; /* non-causal forward apply pass: CTAs per group */
  int32_t full_ctas_bwd; /* non-causal backward pass: CTAs per group */
  int32_t prefetch;      /* L2 prefetch distance (chunks) ahead of the TMA ring */
  int32_t host_blocks;   /* la_host_step: group blocks per step (default 16) */
  int32_t simt_seg_rows; /* CUDA-core path: minimum rows per segment (default 32) */
  int32_t bwd_pair;      /* causal backward as 2-CTA clusters: 1 force, -1 never, 0 rule */
} la_tuning;
void la_set_tuning(const la_tuning* t); /* NULL restores the built-in rules */
void la_get_tuning(la_tuning* t);

/* ---------------------------------------------------------------- queries */
const char* la_version(void);
const char* la_status_name(la_status s);
size_t la_forward_workspace_bytes(const la_problem* p);
size_t la_backward_workspace_bytes(const la_problem* p);
size_t la_shard_state_floats(const la_problem* p); /* G * (D*D + 2*D + 1, padded to 4) */
la_status la_validate_plan(const la_block_plan* plan, int64_t groups, int64_t dim,
                           la_error_info* err);
la_status la_default_plan(int64_t groups, int64_t dim, int32_t workers, la_block_plan* out);
/* Kernel launches issued by this library since load (for bench accounting). */
uint64_t la_launch_count(void);
/* Per-kernel device timing: while enabled, every kernel this library launches
 * is bracketed by CUDA events on its stream. la_profile_read synchronises and
 * writes a JSON array [{"name": ..., "ms": ...}, ...] of the launches since the
 * last read, then clears the list. Returns the number of records. */
void la_profile_enable(int32_t on);
int32_t la_profile_read(char* json, size_t cap);

/* ---------------------------------------------------------------- device API */
la_status la_forward(const la_problem* p, const void* q, la_layout lq, const void* k, la_layout lk,
                     const void* v, la_layout lv, void* out /* FeatureMajor */,
                     float* g /* G*N */, void* workspace, size_t ws_bytes, void* stream,
                     la_error_info* err);

la_status la_backward(const la_problem* p, const void* q, la_layout lq, const void* k,
                      la_layout lk, const void* v, la_layout lv, const void* o /* FeatureMajor */,
                      const void* omega, la_layout lw, const float* g,
                      void* dq /* SequenceMajor */, void* dk /* FeatureMajor */,
                      void* dv /* FeatureMajor */, void* workspace, size_t ws_bytes,
                      void* stream, la_error_info* err);

/* Forward that also saves, per (group, segment), the prefix state at the
 * segment's last row (la_saved_state_bytes(p) bytes, device memory). Handing it
 * to la_backward_saved spares the backward from re-reading K and V for its
 * prefix states, the way ForwardArtifacts carries (out, g) (forward.hpp:35-41).
 * The buffer must come from la_forward_save of the same problem: the library
 * remembers which buffers its forwards wrote (no device read in the backward, so a
 * forward + backward step is stream-asynchronous and CUDA-graph capturable); a buffer
 * it does not know is checked through its header (one synchronising read). */
size_t la_saved_state_bytes(const la_problem* p);
la_status la_forward_save(const la_problem* p, const void* q, la_layout lq, const void* k,
                          la_layout lk, const void* v, la_layout lv, void* out, float* g,
                          void* saved, size_t saved_bytes, void* workspace, size_t ws_bytes,
                          void* stream, la_error_info* err);
la_status la_backward_saved(const la_problem* p, const void* q, la_layout lq, const void* k,
                            la_layout lk, const void* v, la_layout lv, const void* o,
                            const void* omega, la_layout lw, const float* g, const void* saved,
                            size_t saved_bytes, void* dq, void* dk, void* dv, void* workspace,
                            size_t ws_bytes, void* stream, la_error_info* err);

/* Sequence-sharded variants: same as above on one shard, with carries. */
la_status la_forward_sharded(const la_problem* p, const la_shard* shard, const void* q,
                             la_layout lq, const void* k, la_layout lk, const void* v,
                             la_layout lv, void* out, float* g, void* workspace, size_t ws_bytes,
                             void* stream, la_error_info* err);
la_status la_backward_sharded(const la_problem* p, const la_shard* shard, const void* q,
                              la_layout lq, const void* k, la_layout lk, const void* v,
                              la_layout lv, const void* o, const void* omega, la_layout lw,
                              const float* g, void* dq, void* dk, void* dv, void* workspace,
                              size_t ws_bytes, void* stream, la_error_info* err);
/* The same with the forward's per-segment saved states (see la_forward_save): the
 * carried backward then skips its K/V aggregate pass. */
la_status la_forward_sharded_save(const la_problem* p, const la_shard* shard, const void* q, la_layout lq,
                                  const void* k, la_layout lk, const void* v, la_layout lv, void* out, float* g,
                                  void* saved, size_t saved_bytes, void* workspace, size_t ws_bytes, void* stream,
                                  la_error_info* err);
la_status la_backward_sharded_saved(const la_problem* p, const la_shard* shard, const void* q, la_layout lq,
                                    const void* k, la_layout lk, const void* v, la_layout lv, const void* o,
                                    const void* omega, la_layout lw, const float* g, const void* saved,
                                    size_t saved_bytes, void* dq, void* dk, void* dv, void* workspace,
                                    size_t ws_bytes, void* stream, la_error_info* err);
/* Shard totals to exchange: forward (S=sum k^T v, z=sum k, sigma=sum v, count);
 * backward (R=sum q^T w_hat, u=sum s q, c=sum w_hat). Written to `state_out`
 * (la_shard_state_floats(p) fp32 values, device); `workspace` is device scratch of
 * la_shard_state_workspace_bytes(p) bytes. */
size_t la_shard_state_workspace_bytes(const la_problem* p);
la_status la_forward_shard_state(const la_problem* p, const void* k, la_layout lk, const void* v,
                                 la_layout lv, float* state_out, void* workspace, size_t ws_bytes,
                                 void* stream);
la_status la_backward_shard_state(const la_problem* p, const void* q, la_layout lq,
                                  const void* o, const void* omega, la_layout lw, const float* g,
                                  float* state_out, void* workspace, size_t ws_bytes, void* stream);
/* Exclusive prefix (forward) / suffix (backward) of `nshards` gathered shard
 * states for shard `rank`, in fp32 on the device: the local step of the
 * NCCL all-gather scan. */
la_status la_combine_shard_states(const la_problem* p, const float* gathered, int32_t nshards,
                                  int32_t rank, int32_t suffix, float* carry_out, void* stream);

la_status la_query_status(const void* workspace, void* stream, la_error_info* err);

/* ---------------------------------------------------------------- multi-GPU
 * One process per GPU. The reference has no multi-device path; these entries shard
 * the groups-independent work of run_forward / run_backward (forward_kernels.hpp:
 * 221-235, backward_kernels.hpp:292-396) across ranks:
 *   LA_SHARD_BATCH_HEAD  each rank owns whole groups (p->groups = its local count);
 *                        no collective at all.
 *   LA_SHARD_SEQUENCE    each rank owns rows [row_offset, row_offset + p->seq_len) of
 *                        every group (causal). Forward: shard totals (S, z, sigma, rows)
 *                        -> one all-gather -> exclusive prefix as the carry. Backward:
 *                        (R, u, c, rows) -> all-gather -> exclusive suffix.
 * The all-gather is ncclAllGather on `nccl_comm` (an ncclComm_t over the nranks
 * processes, e.g. from la_nccl_comm_init) on the call's stream; when nccl_comm is
 * NULL the caller's `allgather` callback performs it instead (tests use this to run
 * several ranks on one device). */
typedef enum { LA_SHARD_BATCH_HEAD = 0, LA_SHARD_SEQUENCE = 1 } la_shard_mode;
/* recv[r * count .. (r+1) * count) = rank r's send[0 .. count), device fp32 buffers,
 * stream-ordered on `stream`; returns 0 on success. */
typedef int (*la_allgather_fn)(const float* send, float* recv, size_t count, void* ctx, void* stream);
typedef struct {
  la_shard_mode mode;
  int32_t rank, nranks;
  int64_t row_offset;      /* SEQUENCE: global index of this rank's first row */
  void* nccl_comm;         /* ncclComm_t, or NULL to use `allgather` */
  la_allgather_fn allgather;
  void* allgather_ctx;
} la_dist;
/* `saved`: the forward's artifacts for the backward (per-segment states + the
 * forward carry), la_dist_saved_bytes; `workspace`: la_dist_workspace_bytes, for
 * either pass. Both device, caller-owned. */
size_t la_dist_saved_bytes(const la_problem* p, const la_dist* d);
size_t la_dist_workspace_bytes(const la_problem* p, const la_dist* d);
la_status la_sharded_forward(const la_problem* p, const la_dist* d, const void* q, la_layout lq, const void* k,
                             la_layout lk, const void* v, la_layout lv, void* out, float* g, void* saved,
                             size_t saved_bytes, void* workspace, size_t ws_bytes, void* stream,
                             la_error_info* err);
la_status la_sharded_backward(const la_problem* p, const la_dist* d, const void* q, la_layout lq, const void* k,
                              la_layout lk, const void* v, la_layout lv, const void* o, const void* omega,
                              la_layout lw, const float* g, const void* saved, size_t saved_bytes, void* dq,
                              void* dk, void* dv, void* workspace, size_t ws_bytes, void* stream,
                              la_error_info* err);
/* NCCL bootstrap without linking NCCL into the caller (libnccl.so.2 is loaded at
 * first use; LA_ERR_UNSUPPORTED when absent). id: 128 bytes (ncclUniqueId). */
la_status la_nccl_get_unique_id(char* id);
la_status la_nccl_comm_init(void** comm, int32_t nranks, const char* id, int32_t rank);
la_status la_nccl_comm_destroy(void* comm);

/* ------------------------------------------- input prologue and diagnostics (device)
 * The reference's API calls either side of the hot path.
 * Tensors are (G, N, D) in p->dtype; accumulators are the reference's TermAccumulator
 * (forward.hpp:44-50): FeatureMajor G*N*D, fp32 on the device. */
/* normalize_qk (plan.cpp:95-117): every row scaled to unit L2 norm, zero rows left as
 * they are; outputs keep the input layouts and may alias the inputs. */
la_status la_normalize_qk(const la_problem* p, const void* q, la_layout lq, const void* k, la_layout lk,
                          void* q_out, void* k_out, void* stream, la_error_info* err);
/* relayout (tensor.cpp:101-119): copy of x in layout ly. */
la_status la_relayout(const la_problem* p, const void* x, la_layout lx, void* y, la_layout ly, void* stream,
                      la_error_info* err);
/* make_omega_hat (backward.cpp:74-91): out = omega / g per row, FeatureMajor. */
la_status la_make_omega_hat(const la_problem* p, const void* omega, la_layout lw, const float* g, void* out,
                            void* stream, la_error_info* err);
/* constant_term_pass (forward.cpp:97-107): f_ij = a * sum_{n<=i} v_nj (overwrites f). */
la_status la_constant_term_pass(const la_problem* p, const void* v, la_layout lv, float* f, void* stream,
                                la_error_info* err);
/* linear_term_pass (forward.cpp:109-131): f_ij += sum_m q_im * b * sum_{n<=i} k_nm v_nj. */
la_status la_linear_term_pass(const la_problem* p, const void* q, la_layout lq, const void* k, la_layout lk,
                              const void* v, la_layout lv, float* f, void* stream, la_error_info* err);
/* alpha_term_pass (backward.cpp:103-128), b = p->b: dk_ir = sum_j alphaK_rj v_ij with
 * alphaK_rj = b * sum_{t>=i} q_tr * omega_hat_tj (overwrites dk). */
la_status la_alpha_term_pass(const la_problem* p, const void* q, la_layout lq, const void* v, la_layout lv,
                             const void* omega_hat, la_layout lw, float* dk, void* stream, la_error_info* err);
/* beta_term_pass (backward.cpp:130-153), b = p->b: dk_ir -= b * sum_{t>=i} q_tr * sum_j o_tj omega_hat_tj. */
la_status la_beta_term_pass(const la_problem* p, const void* q, la_layout lq, const void* o, la_layout lo,
                            const void* omega_hat, la_layout lw, float* dk, void* stream, la_error_info* err);

/* ---------------------------------------------------------------- host API */
/* End-to-end over host buffers: copies inputs to the device, runs, copies the
 * results back (device arena cached per thread). Used by the reference-facing
 * shim and the e2e bench. */
la_status la_host_forward(const la_problem* p, const void* q, la_layout lq, const void* k,
                          la_layout lk, const void* v, la_layout lv, void* out, float* g,
                          la_error_info* err);
la_status la_host_backward(const la_problem* p, const void* q, la_layout lq, const void* k,
                           la_layout lk, const void* v, la_layout lv, const void* o,
                           const void* omega, la_layout lw, const float* g, void* dq, void* dk,
                           void* dv, la_error_info* err);
/* One training step over host buffers: forward_causal/forward_full followed by
 * backward_causal/backward_full on the same inputs (forward.cpp:133-142,
 * backward.cpp:93-101, as bench.cpp:137-139 + :176-179 time them). Inputs q, k, v,
 * omega are copied in once and out, g, dq, dk, dv copied back; the groups are
 * processed in blocks so host->device copies, compute and device->host copies
 * overlap (pinned host memory gives the full PCIe rate in both directions). */
la_status la_host_step(const la_problem* p, const void* q, la_layout lq, const void* k,
                       la_layout lk, const void* v, la_layout lv, const void* omega, la_layout lw,
                       void* out, float* g, void* dq, void* dk, void* dv, la_error_info* err);
void la_host_release(void);

#ifdef __cplusplus
}
#endif
#endif /* LA_CUDA_H */
