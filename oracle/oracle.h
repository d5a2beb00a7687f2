/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the linear-attention path.
 *
 * A plain-C restatement of the reference library's CPU kernels
 * (/root/reference/proj/include/la/detail/forward_kernels.hpp and
 * backward_kernels.hpp), loop for loop, at plan L=1 (one work item per
 * group owning every feature; the reference proves its outputs are bitwise
 * identical across L, verify.cpp:230-279). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this; the
 * product path (paper_2510_21956_b200/) never links or calls it.
 *
 * Parity is PINNED: the restatement reproduces the reference's own goldens
 * (tests/test_forward.cpp:115-134, tests/test_backward.cpp:74-113) and is
 * cross-checked element-for-element against the reference sources compiled
 * into oracle/_ref/libla_ref.so (see oracle/Makefile, tests/test_oracle.py).
 *
 * Layout codes follow la::Layout (tensor.hpp:15): 0 = FeatureMajor
 * (g*N*D + j*N + i), 1 = SequenceMajor (g*N*D + i*D + j).
 * Fault codes follow la::Fault (fault.hpp:7-15).
 * Return value: 0 on success, 1 + (index of the first degenerate row) encoded
 * through *bad_group / *bad_pos (DegenerateDenominator, forward_kernels.hpp:53).
 */
#ifndef LA_ORACLE_H
#define LA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* std::mt19937_64 seeded fill in logical (g,i,j) order (tensor.cpp:43-77). */
void oracle_fill_uniform(double* out, int64_t groups, int64_t n, int64_t d, int layout,
                         uint64_t seed, double lo, double hi);
/* Row-wise Euclidean normalisation, zero rows untouched (plan.cpp:95-117). */
void oracle_normalize_rows(double* data, int64_t groups, int64_t n, int64_t d, int layout);

/* la::detail::run_forward<T> (forward_kernels.hpp:210-259).  out is FeatureMajor. */
int oracle_forward_f64(const double* q, int lq, const double* k, int lk, const double* v, int lv,
                       int64_t groups, int64_t n, int64_t d, double a, double b, int causal,
                       int fault, double* out, double* g, int64_t* bad_group, int64_t* bad_pos);
int oracle_forward_f32(const float* q, int lq, const float* k, int lk, const float* v, int lv,
                       int64_t groups, int64_t n, int64_t d, double a, double b, int causal,
                       int fault, float* out, float* g, int64_t* bad_group, int64_t* bad_pos);

/* la::detail::run_backward<T> (backward_kernels.hpp:292-396).
 * o is the forward output (layout lo), dq SequenceMajor, dk/dv FeatureMajor. */
void oracle_backward_f64(const double* q, int lq, const double* k, int lk, const double* v,
                         int lv, const double* o, int lo, const double* omega, int lw,
                         const double* g, int64_t groups, int64_t n, int64_t d, double a,
                         double b, int causal, int fault, double* dq, double* dk, double* dv);
void oracle_backward_f32(const float* q, int lq, const float* k, int lk, const float* v, int lv,
                         const float* o, int lo, const float* omega, int lw, const float* g,
                         int64_t groups, int64_t n, int64_t d, double a, double b, int causal,
                         int fault, float* dq, float* dk, float* dv);

/* Brute-force O(N^2 D) ground truth (reference.cpp:67-106); out SequenceMajor. */
int oracle_quadratic(const double* q, int lq, const double* k, int lk, const double* v, int lv,
                     int64_t groups, int64_t n, int64_t d, double a, double b, int causal,
                     double* out, double* g, int64_t* bad_group, int64_t* bad_pos);

/* Multi-threaded f32 timing harness used by the CPU baseline: the same
 * per-group restatement run over `threads` std-C threads (bench.cpp:111-191
 * times run_forward<float> + run_backward<float> with workers = nproc). */
int oracle_fwd_bwd_f32_threads(const float* q, const float* k, const float* v,
                               const float* omega, int64_t groups, int64_t n, int64_t d,
                               double a, double b, int causal, int threads, float* out,
                               float* g, float* dq, float* dk, float* dv);

#ifdef __cplusplus
}
#endif
#endif
