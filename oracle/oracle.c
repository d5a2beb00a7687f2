/*
 * TEST INFRASTRUCTURE ONLY — see oracle.h. CPU restatement of the reference
 * linear-attention kernels, used as the parity checker and as the CPU-baseline
 * fallback ("kind": "port"). Never linked by the product library.
 *
 * Each function cites the reference loop it restates. Arithmetic is kept in
 * the template type T exactly as the reference does (a and b are cast to T
 * first, forward_kernels.hpp:215-216), so f32 results match the reference's
 * run_forward<float> / run_backward<float> bit for bit when both are built
 * without FMA contraction (see oracle/Makefile).
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the generator make_tensor uses, tensor.cpp:60).          */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
typedef struct {
  uint64_t mt[MT_N];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = MT_N;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (s->idx >= MT_N) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_N - MT_M; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + MT_M] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    for (; i < MT_N - 1; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    }
    x = (s->mt[MT_N - 1] & UM) | (s->mt[0] & LM);
    s->mt[MT_N - 1] = s->mt[MT_M - 1] ^ (x >> 1) ^ mag[(int)(x & 1ULL)];
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* tensor.cpp:35-41 */
static inline size_t flat_index(int64_t g, int64_t i, int64_t j, int64_t n, int64_t d,
                                int layout) {
  const size_t base = (size_t)g * (size_t)n * (size_t)d;
  if (layout == 0) return base + (size_t)j * (size_t)n + (size_t)i;
  return base + (size_t)i * (size_t)d + (size_t)j;
}

/* tensor.cpp:14-16, 58-72 */
void oracle_fill_uniform(double* out, int64_t groups, int64_t n, int64_t d, int layout,
                         uint64_t seed, double lo, double hi) {
  mt64* s = (mt64*)malloc(sizeof(mt64));
  mt64_seed(s, seed);
  const double width = hi - lo;
  for (int64_t g = 0; g < groups; ++g)
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < d; ++j)
        out[flat_index(g, i, j, n, d, layout)] =
            lo + width * ((double)(mt64_next(s) >> 11) * 0x1.0p-53);
  free(s);
}

/* plan.cpp:95-117 */
void oracle_normalize_rows(double* data, int64_t groups, int64_t n, int64_t d, int layout) {
  for (int64_t g = 0; g < groups; ++g) {
    for (int64_t i = 0; i < n; ++i) {
      double sq = 0.0;
      for (int64_t j = 0; j < d; ++j) {
        const double x = data[flat_index(g, i, j, n, d, layout)];
        sq += x * x;
      }
      if (sq == 0.0) continue;
      const double inv = 1.0 / sqrt(sq);
      for (int64_t j = 0; j < d; ++j) data[flat_index(g, i, j, n, d, layout)] *= inv;
    }
  }
}

/* Strided (istride, jstride) per layout, view.hpp:46-55. */
#define STRIDES(layout, n, d, is, js) \
  do {                                \
    if ((layout) == 0) {              \
      is = 1;                         \
      js = (size_t)(n);               \
    } else {                          \
      is = (size_t)(d);               \
      js = 1;                         \
    }                                 \
  } while (0)

/* ------------------------------------------------------------------------ */
/* Forward: forward_kernels.hpp, instantiated for T = double and T = float.  */
/* ------------------------------------------------------------------------ */
#define DEFINE_FORWARD(T, SUF, EPS, FABS)                                                         \
  int oracle_forward_##SUF(const T* q, int lq, const T* k, int lk, const T* v, int lv,            \
                           int64_t groups, int64_t n, int64_t d, double a_, double b_,           \
                           int causal, int fault, T* out, T* g_vec, int64_t* bad_group,          \
                           int64_t* bad_pos) {                                                   \
    const T a = (T)a_, b = (T)b_, eps = (EPS);                                                   \
    size_t qi, qj, ki, kj, vi, vj;                                                               \
    STRIDES(lq, n, d, qi, qj);                                                                   \
    STRIDES(lk, n, d, ki, kj);                                                                   \
    STRIDES(lv, n, d, vi, vj);                                                                   \
    const size_t gsz = (size_t)n * (size_t)d;                                                    \
    T* y2 = (T*)calloc((size_t)d, sizeof(T));                                                    \
    T* x1 = (T*)calloc((size_t)d, sizeof(T));                                                    \
    T* x2 = (T*)calloc((size_t)d * (size_t)d, sizeof(T));                                        \
    T* qs = (T*)calloc((size_t)d, sizeof(T));                                                    \
    T* ks = (T*)calloc((size_t)d, sizeof(T));                                                    \
    int status = 0;                                                                              \
    /* Phase "forward.constant" (forward_kernels.hpp:218-236): every group, in item order. */   \
    for (int64_t grp = 0; grp < groups && !status; ++grp) {                                      \
      const T* qg = q + grp * gsz;                                                               \
      const T* kg = k + grp * gsz;                                                               \
      const T* vg = v + grp * gsz;                                                               \
      T* f = out + grp * gsz;                                                                    \
      T* gr = g_vec + grp * n;                                                                   \
      memset(y2, 0, sizeof(T) * (size_t)d);                                                      \
      if (causal) {                                                                              \
        /* constant_causal_core :22-34 */                                                        \
        for (int64_t j = 0; j < d; ++j) {                                                        \
          T acc = (T)0;                                                                          \
          for (int64_t i = 0; i < n; ++i) {                                                      \
            acc += a * vg[(size_t)i * vi + (size_t)j * vj];                                      \
            f[(size_t)j * n + i] = acc;                                                          \
          }                                                                                      \
        }                                                                                        \
        /* denominator_causal_core :38-56 */                                                     \
        for (int64_t i = 0; i < n; ++i) {                                                        \
          T acc = a * (T)(i + 1);                                                                \
          for (int64_t m = 0; m < d; ++m) {                                                      \
            y2[m] += b * kg[(size_t)i * ki + (size_t)m * kj];                                    \
            acc += qg[(size_t)i * qi + (size_t)m * qj] * y2[m];                                  \
          }                                                                                      \
          if (FABS(acc) < eps) {                                                                 \
            *bad_group = grp;                                                                    \
            *bad_pos = i;                                                                        \
            status = 1;                                                                          \
            break;                                                                               \
          }                                                                                      \
          gr[i] = acc;                                                                           \
        }                                                                                        \
      } else {                                                                                   \
        /* constant_full_core :133-146 */                                                        \
        for (int64_t j = 0; j < d; ++j) {                                                        \
          T acc = (T)0;                                                                          \
          for (int64_t i = 0; i < n; ++i) acc += a * vg[(size_t)i * vi + (size_t)j * vj];        \
          x1[j] = acc;                                                                           \
          for (int64_t i = 0; i < n; ++i) f[(size_t)j * n + i] = acc;                            \
        }                                                                                        \
        /* denominator_full_core :148-167 */                                                     \
        for (int64_t i = 0; i < n; ++i)                                                          \
          for (int64_t m = 0; m < d; ++m) y2[m] += b * kg[(size_t)i * ki + (size_t)m * kj];      \
        const T base = a * (T)n;                                                                 \
        for (int64_t i = 0; i < n; ++i) {                                                        \
          T acc = base;                                                                          \
          for (int64_t m = 0; m < d; ++m) acc += qg[(size_t)i * qi + (size_t)m * qj] * y2[m];    \
          if (FABS(acc) < eps) {                                                                 \
            *bad_group = grp;                                                                    \
            *bad_pos = i;                                                                        \
            status = 1;                                                                          \
            break;                                                                               \
          }                                                                                      \
          gr[i] = acc;                                                                           \
        }                                                                                        \
      }                                                                                          \
    }                                                                                            \
    /* Phase "forward.linear" (forward_kernels.hpp:238-258), only if phase 1 succeeded. */      \
    for (int64_t grp = 0; grp < groups && !status; ++grp) {                                      \
      const T* qg = q + grp * gsz;                                                               \
      const T* kg = k + grp * gsz;                                                               \
      const T* vg = v + grp * gsz;                                                               \
      T* f = out + grp * gsz;                                                                    \
      const T* gr = g_vec + grp * n;                                                             \
      memset(x2, 0, sizeof(T) * (size_t)d * (size_t)d);                                          \
      if (causal && fault == 2) {                                                                \
        /* CausalPrefixOffByOne branch, linear_causal_core :86-106 */                            \
        int64_t absorbed = 0;                                                                    \
        for (int64_t i = 0; i < n; ++i) {                                                        \
          const int64_t want = i + 1 < n ? i + 1 : n - 1;                                        \
          while (absorbed <= want) {                                                             \
            const int64_t row = absorbed++;                                                      \
            for (int64_t m = 0; m < d; ++m) ks[m] = b * kg[(size_t)row * ki + (size_t)m * kj];   \
            for (int64_t j = 0; j < d; ++j) {                                                    \
              const T vij = vg[(size_t)row * vi + (size_t)j * vj];                               \
              T* st = x2 + (size_t)j * d;                                                        \
              for (int64_t m = 0; m < d; ++m) st[m] += ks[m] * vij;                              \
            }                                                                                    \
          }                                                                                      \
          for (int64_t m = 0; m < d; ++m) qs[m] = qg[(size_t)i * qi + (size_t)m * qj];           \
          for (int64_t j = 0; j < d; ++j) {                                                      \
            const T* st = x2 + (size_t)j * d;                                                    \
            T acc = (T)0;                                                                        \
            for (int64_t m = 0; m < d; ++m) acc += qs[m] * st[m];                                \
            T* slot = f + (size_t)j * n + i;                                                     \
            const T val = *slot + acc;                                                           \
            *slot = val / gr[i];                                                                 \
          }                                                                                      \
        }                                                                                        \
      } else if (causal) {                                                                       \
        /* linear_causal_core hot loop :108-127 */                                               \
        for (int64_t i = 0; i < n; ++i) {                                                        \
          for (int64_t m = 0; m < d; ++m) {                                                      \
            qs[m] = qg[(size_t)i * qi + (size_t)m * qj];                                         \
            ks[m] = b * kg[(size_t)i * ki + (size_t)m * kj];                                     \
          }                                                                                      \
          for (int64_t j = 0; j < d; ++j) {                                                      \
            const T vij = vg[(size_t)i * vi + (size_t)j * vj];                                   \
            T* st = x2 + (size_t)j * d;                                                          \
            T acc = (T)0;                                                                        \
            for (int64_t m = 0; m < d; ++m) {                                                    \
              st[m] += ks[m] * vij;                                                              \
              acc += qs[m] * st[m];                                                              \
            }                                                                                    \
            T* slot = f + (size_t)j * n + i;                                                     \
            const T val = *slot + acc;                                                           \
            *slot = val / gr[i];                                                                 \
          }                                                                                      \
        }                                                                                        \
      } else {                                                                                   \
        /* linear_full_core :170-206 */                                                          \
        for (int64_t i = 0; i < n; ++i) {                                                        \
          for (int64_t m = 0; m < d; ++m) ks[m] = b * kg[(size_t)i * ki + (size_t)m * kj];      \
          for (int64_t j = 0; j < d; ++j) {                                                      \
            const T vij = vg[(size_t)i * vi + (size_t)j * vj];                                   \
            T* st = x2 + (size_t)j * d;                                                          \
            for (int64_t m = 0; m < d; ++m) st[m] += ks[m] * vij;                                \
          }                                                                                      \
        }                                                                                        \
        for (int64_t i = 0; i < n; ++i) {                                                        \
          for (int64_t m = 0; m < d; ++m) qs[m] = qg[(size_t)i * qi + (size_t)m * qj];           \
          for (int64_t j = 0; j < d; ++j) {                                                      \
            const T* st = x2 + (size_t)j * d;                                                    \
            T acc = (T)0;                                                                        \
            for (int64_t m = 0; m < d; ++m) acc += qs[m] * st[m];                                \
            T* slot = f + (size_t)j * n + i;                                                     \
            const T val = *slot + acc;                                                           \
            *slot = val / gr[i];                                                                 \
          }                                                                                      \
        }                                                                                        \
      }                                                                                          \
    }                                                                                            \
    free(y2);                                                                                    \
    free(x1);                                                                                    \
    free(x2);                                                                                    \
    free(qs);                                                                                    \
    free(ks);                                                                                    \
    return status;                                                                               \
  }

static inline double fabs_d(double x) { return fabs(x); }
static inline float fabs_f(float x) { return fabsf(x); }
DEFINE_FORWARD(double, f64, 1e-8, fabs_d)
DEFINE_FORWARD(float, f32, 1e-4f, fabs_f)

/* ------------------------------------------------------------------------ */
/* Backward: backward_kernels.hpp, per group, L = 1 (r0 = 0, r1 = D).        */
/* ------------------------------------------------------------------------ */
#define DEFINE_BACKWARD_GROUP(T, SUF)                                                             \
  static void backward_group_##SUF(                                                               \
      const T* qg, size_t qi, size_t qj, const T* kg, size_t ki, size_t kj, const T* vg,          \
      size_t vi, size_t vj, const T* og, size_t oi, size_t oj, const T* wg, size_t wi, size_t wj, \
      const T* gr, int64_t n, int64_t d, T a, T b, int causal, int fault, T* dqg, T* dkg,         \
      T* dvg) {                                                                                   \
    /* dq SequenceMajor, dk/dv FeatureMajor (backward.cpp:42-44). */                             \
    const size_t dd = (size_t)d * (size_t)d;                                                      \
    T* alpha = (T*)calloc(dd, sizeof(T));                                                         \
    T* beta = (T*)calloc(dd, sizeof(T));                                                          \
    T* vrow = (T*)calloc((size_t)d, sizeof(T));                                                   \
    T* whrow = (T*)calloc((size_t)d, sizeof(T));                                                  \
    T* kb = (T*)calloc((size_t)d, sizeof(T));                                                     \
    T* bvec = (T*)calloc((size_t)d, sizeof(T));                                                   \
    const int flip = fault == 1, drop = fault == 3;                                               \
    if (causal) {                                                                                 \
      /* grad_q_causal_core :21-57 */                                                             \
      for (int64_t i = 0; i < n; ++i) {                                                           \
        const T gi = gr[i];                                                                       \
        T s = (T)0;                                                                               \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          vrow[j] = vg[(size_t)i * vi + (size_t)j * vj];                                          \
          whrow[j] = wg[(size_t)i * wi + (size_t)j * wj] / gi;                                    \
          s += og[(size_t)i * oi + (size_t)j * oj] * whrow[j];                                    \
        }                                                                                         \
        for (int64_t r = 0; r < d; ++r) kb[r] = b * kg[(size_t)i * ki + (size_t)r * kj];          \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T kr = kb[r];                                                                     \
          T* arow = alpha + (size_t)r * d;                                                        \
          for (int64_t j = 0; j < d; ++j) arow[j] += kr * vrow[j];                                \
          bvec[r] += kr;                                                                          \
        }                                                                                         \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T* arow = alpha + (size_t)r * d;                                                  \
          T acc = (T)0;                                                                           \
          for (int64_t j = 0; j < d; ++j) acc += arow[j] * whrow[j];                              \
          dqg[(size_t)i * d + r] = acc - bvec[r] * s;                                             \
        }                                                                                         \
      }                                                                                           \
      /* grad_k_alpha_core :61-91 (assigns dk) */                                                 \
      memset(alpha, 0, dd * sizeof(T));                                                           \
      for (int64_t i = n - 1; i >= 0; --i) {                                                      \
        const T gi = gr[i];                                                                       \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          vrow[j] = vg[(size_t)i * vi + (size_t)j * vj];                                          \
          whrow[j] = wg[(size_t)i * wi + (size_t)j * wj] / gi;                                    \
        }                                                                                         \
        for (int64_t r = 0; r < d; ++r) kb[r] = b * qg[(size_t)i * qi + (size_t)r * qj];          \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T qr = kb[r];                                                                     \
          T* arow = alpha + (size_t)r * d;                                                        \
          T acc = (T)0;                                                                           \
          for (int64_t j = 0; j < d; ++j) {                                                       \
            arow[j] += qr * whrow[j];                                                             \
            acc += arow[j] * vrow[j];                                                             \
          }                                                                                       \
          dkg[(size_t)r * n + i] = acc;                                                           \
        }                                                                                         \
      }                                                                                           \
      /* grad_k_beta_core :95-130 (subtracts from dk) */                                          \
      memset(beta, 0, dd * sizeof(T));                                                            \
      for (int64_t i = n - 1; i >= 0; --i) {                                                      \
        const T gi = gr[i];                                                                       \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          const T wh = wg[(size_t)i * wi + (size_t)j * wj] / gi;                                  \
          whrow[j] = og[(size_t)i * oi + (size_t)j * oj] * wh; /* powrow */                       \
        }                                                                                         \
        for (int64_t r = 0; r < d; ++r) kb[r] = b * qg[(size_t)i * qi + (size_t)r * qj];          \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T qr = kb[r];                                                                     \
          T* brow = beta + (size_t)r * d;                                                         \
          T acc = (T)0;                                                                           \
          for (int64_t j = 0; j < d; ++j) {                                                       \
            brow[j] += qr * whrow[j];                                                             \
            acc += brow[j];                                                                       \
          }                                                                                       \
          if (flip)                                                                               \
            dkg[(size_t)r * n + i] += acc;                                                        \
          else                                                                                    \
            dkg[(size_t)r * n + i] -= acc;                                                        \
        }                                                                                         \
      }                                                                                           \
      /* grad_v_causal_core :134-168 */                                                           \
      memset(beta, 0, dd * sizeof(T));                                                            \
      memset(bvec, 0, (size_t)d * sizeof(T));                                                     \
      for (int64_t i = n - 1; i >= 0; --i) {                                                      \
        const T gi = gr[i];                                                                       \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          kb[r] = b * qg[(size_t)i * qi + (size_t)r * qj]; /* qb */                               \
          vrow[r] = kg[(size_t)i * ki + (size_t)r * kj];   /* krow */                             \
        }                                                                                         \
        for (int64_t j = 0; j < d; ++j) whrow[j] = wg[(size_t)i * wi + (size_t)j * wj] / gi;      \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          const T wh = whrow[j];                                                                  \
          bvec[j] += a * wh; /* alpha_v */                                                        \
          T* brow = beta + (size_t)j * d;                                                         \
          T acc = (T)0;                                                                           \
          for (int64_t r = 0; r < d; ++r) {                                                       \
            brow[r] += kb[r] * wh;                                                                \
            acc += vrow[r] * brow[r];                                                             \
          }                                                                                       \
          dvg[(size_t)j * n + i] = drop ? acc : bvec[j] + acc;                                    \
        }                                                                                         \
      }                                                                                           \
    } else {                                                                                      \
      /* grad_q_full_core :173-208 */                                                             \
      for (int64_t l = 0; l < n; ++l) {                                                           \
        for (int64_t j = 0; j < d; ++j) vrow[j] = vg[(size_t)l * vi + (size_t)j * vj];            \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T kr = b * kg[(size_t)l * ki + (size_t)r * kj];                                   \
          T* arow = alpha + (size_t)r * d;                                                        \
          for (int64_t j = 0; j < d; ++j) arow[j] += kr * vrow[j];                                \
          bvec[r] += kr;                                                                          \
        }                                                                                         \
      }                                                                                           \
      for (int64_t i = 0; i < n; ++i) {                                                           \
        const T gi = gr[i];                                                                       \
        T s = (T)0;                                                                               \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          whrow[j] = wg[(size_t)i * wi + (size_t)j * wj] / gi;                                    \
          s += og[(size_t)i * oi + (size_t)j * oj] * whrow[j];                                    \
        }                                                                                         \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T* arow = alpha + (size_t)r * d;                                                  \
          T acc = (T)0;                                                                           \
          for (int64_t j = 0; j < d; ++j) acc += arow[j] * whrow[j];                              \
          dqg[(size_t)i * d + r] = acc - bvec[r] * s;                                             \
        }                                                                                         \
      }                                                                                           \
      /* grad_k_full_core :210-248 */                                                             \
      memset(alpha, 0, dd * sizeof(T));                                                           \
      memset(bvec, 0, (size_t)d * sizeof(T));                                                     \
      for (int64_t i = 0; i < n; ++i) {                                                           \
        const T gi = gr[i];                                                                       \
        T s = (T)0;                                                                               \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          whrow[j] = wg[(size_t)i * wi + (size_t)j * wj] / gi;                                    \
          s += og[(size_t)i * oi + (size_t)j * oj] * whrow[j];                                    \
        }                                                                                         \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T qr = b * qg[(size_t)i * qi + (size_t)r * qj];                                   \
          T* arow = alpha + (size_t)r * d;                                                        \
          for (int64_t j = 0; j < d; ++j) arow[j] += qr * whrow[j];                               \
          bvec[r] += qr * s;                                                                      \
        }                                                                                         \
      }                                                                                           \
      for (int64_t p = 0; p < n; ++p) {                                                           \
        for (int64_t j = 0; j < d; ++j) vrow[j] = vg[(size_t)p * vi + (size_t)j * vj];            \
        for (int64_t r = 0; r < d; ++r) {                                                         \
          const T* arow = alpha + (size_t)r * d;                                                  \
          T acc = (T)0;                                                                           \
          for (int64_t j = 0; j < d; ++j) acc += arow[j] * vrow[j];                               \
          dkg[(size_t)r * n + p] = flip ? acc + bvec[r] : acc - bvec[r];                          \
        }                                                                                         \
      }                                                                                           \
      /* grad_v_full_core :250-288 */                                                             \
      memset(beta, 0, dd * sizeof(T));                                                            \
      memset(bvec, 0, (size_t)d * sizeof(T));                                                     \
      for (int64_t i = 0; i < n; ++i) {                                                           \
        const T gi = gr[i];                                                                       \
        for (int64_t r = 0; r < d; ++r) kb[r] = b * qg[(size_t)i * qi + (size_t)r * qj];          \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          const T wh = wg[(size_t)i * wi + (size_t)j * wj] / gi;                                  \
          bvec[j] += a * wh;                                                                      \
          T* brow = beta + (size_t)j * d;                                                         \
          for (int64_t r = 0; r < d; ++r) brow[r] += kb[r] * wh;                                  \
        }                                                                                         \
      }                                                                                           \
      for (int64_t p = 0; p < n; ++p) {                                                           \
        for (int64_t r = 0; r < d; ++r) vrow[r] = kg[(size_t)p * ki + (size_t)r * kj];            \
        for (int64_t j = 0; j < d; ++j) {                                                         \
          const T* brow = beta + (size_t)j * d;                                                   \
          T acc = (T)0;                                                                           \
          for (int64_t r = 0; r < d; ++r) acc += vrow[r] * brow[r];                               \
          dvg[(size_t)j * n + p] = drop ? acc : bvec[j] + acc;                                    \
        }                                                                                         \
      }                                                                                           \
    }                                                                                             \
    free(alpha);                                                                                  \
    free(beta);                                                                                   \
    free(vrow);                                                                                   \
    free(whrow);                                                                                  \
    free(kb);                                                                                     \
    free(bvec);                                                                                   \
  }                                                                                               \
  void oracle_backward_##SUF(const T* q, int lq, const T* k, int lk, const T* v, int lv,          \
                             const T* o, int lo, const T* omega, int lw, const T* g,              \
                             int64_t groups, int64_t n, int64_t d, double a, double b,            \
                             int causal, int fault, T* dq, T* dk, T* dv) {                        \
    size_t qi, qj, ki, kj, vi, vj, oi, oj, wi, wj;                                                \
    STRIDES(lq, n, d, qi, qj);                                                                    \
    STRIDES(lk, n, d, ki, kj);                                                                    \
    STRIDES(lv, n, d, vi, vj);                                                                    \
    STRIDES(lo, n, d, oi, oj);                                                                    \
    STRIDES(lw, n, d, wi, wj);                                                                    \
    const size_t gsz = (size_t)n * (size_t)d;                                                     \
    for (int64_t grp = 0; grp < groups; ++grp)                                                    \
      backward_group_##SUF(q + grp * gsz, qi, qj, k + grp * gsz, ki, kj, v + grp * gsz, vi, vj,   \
                           o + grp * gsz, oi, oj, omega + grp * gsz, wi, wj, g + grp * n, n, d,   \
                           (T)a, (T)b, causal, fault, dq + grp * gsz, dk + grp * gsz,             \
                           dv + grp * gsz);                                                       \
  }

DEFINE_BACKWARD_GROUP(double, f64)
DEFINE_BACKWARD_GROUP(float, f32)

/* reference.cpp:67-106 */
int oracle_quadratic(const double* q, int lq, const double* k, int lk, const double* v, int lv,
                     int64_t groups, int64_t n, int64_t d, double a, double b, int causal,
                     double* out, double* g_vec, int64_t* bad_group, int64_t* bad_pos) {
  double* row_acc = (double*)calloc((size_t)d, sizeof(double));
  int status = 0;
  for (int64_t g = 0; g < groups && !status; ++g) {
    for (int64_t i = 0; i < n; ++i) {
      const int64_t limit = causal ? i + 1 : n;
      for (int64_t j = 0; j < d; ++j) row_acc[j] = 0.0;
      double denom = 0.0;
      for (int64_t t = 0; t < limit; ++t) {
        double dot = 0.0;
        for (int64_t m = 0; m < d; ++m)
          dot += q[flat_index(g, i, m, n, d, lq)] * k[flat_index(g, t, m, n, d, lk)];
        const double weight = a + b * dot;
        denom += weight;
        for (int64_t j = 0; j < d; ++j) row_acc[j] += weight * v[flat_index(g, t, j, n, d, lv)];
      }
      if (fabs(denom) < 1e-8) {
        *bad_group = g;
        *bad_pos = i;
        status = 1;
        break;
      }
      g_vec[(size_t)g * n + i] = denom;
      for (int64_t j = 0; j < d; ++j) out[(size_t)g * n * d + (size_t)i * d + j] = row_acc[j] / denom;
    }
  }
  free(row_acc);
  return status;
}

/* ------------------------------------------------------------------------ */
/* Threaded f32 fwd+bwd over groups (CPU-baseline port of bench.cpp:111-191: */
/* canonical layouts q,k SequenceMajor, v,omega FeatureMajor).               */
/* ------------------------------------------------------------------------ */
typedef struct {
  const float *q, *k, *v, *omega;
  int64_t n, d, g0, g1;
  double a, b;
  int causal;
  float *out, *g, *dq, *dk, *dv;
  int status;
} job_t;

static void* run_job(void* p) {
  job_t* j = (job_t*)p;
  const size_t gsz = (size_t)j->n * (size_t)j->d;
  int64_t bg, bp;
  for (int64_t grp = j->g0; grp < j->g1; ++grp) {
    const size_t off = (size_t)grp * gsz;
    if (oracle_forward_f32(j->q + off, 1, j->k + off, 1, j->v + off, 0, 1, j->n, j->d, j->a, j->b,
                           j->causal, 0, j->out + off, j->g + (size_t)grp * j->n, &bg, &bp)) {
      j->status = 1;
      return NULL;
    }
    oracle_backward_f32(j->q + off, 1, j->k + off, 1, j->v + off, 0, j->out + off, 0,
                        j->omega + off, 0, j->g + (size_t)grp * j->n, 1, j->n, j->d, j->a, j->b,
                        j->causal, 0, j->dq + off, j->dk + off, j->dv + off);
  }
  return NULL;
}

int oracle_fwd_bwd_f32_threads(const float* q, const float* k, const float* v,
                               const float* omega, int64_t groups, int64_t n, int64_t d,
                               double a, double b, int causal, int threads, float* out,
                               float* g, float* dq, float* dk, float* dv) {
  if (threads < 1) threads = 1;
  if (threads > groups) threads = (int)groups;
  pthread_t* tid = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  for (int t = 0; t < threads; ++t) {
    job_t* j = &jobs[t];
    j->q = q; j->k = k; j->v = v; j->omega = omega;
    j->n = n; j->d = d; j->a = a; j->b = b; j->causal = causal;
    j->g0 = groups * t / threads;
    j->g1 = groups * (t + 1) / threads;
    j->out = out; j->g = g; j->dq = dq; j->dk = dk; j->dv = dv;
    pthread_create(&tid[t], NULL, run_job, j);
  }
  int status = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    status |= jobs[t].status;
  }
  free(tid);
  free(jobs);
  return status;
}
