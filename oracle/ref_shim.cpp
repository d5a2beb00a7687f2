// TEST INFRASTRUCTURE ONLY — a C-ABI shim over the UNMODIFIED reference
// library, compiled from its sources where they lie under /root/reference
// (oracle/Makefile) into oracle/_ref/libla_ref.so. It lets the Python tests
// check the C restatement (oracle.c) against the reference itself and lets
// bench.py time the reference's own CPU path (detail::run_forward<float> /
// run_backward<float>, exactly what bench.cpp:137-139,176-179 times).
// Nothing in the product links this file.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <fstream>

#include "la/backward.hpp"
#include "la/bench.hpp"
#include "la/detail/backward_kernels.hpp"
#include "la/detail/forward_kernels.hpp"
#include "la/detail/view.hpp"
#include "la/forward.hpp"
#include "la/plan.hpp"
#include "la/reference.hpp"
#include "la/tensor.hpp"

namespace {

la::Layout lay(int l) { return l == 0 ? la::Layout::FeatureMajor : la::Layout::SequenceMajor; }
la::Fault fault_of(int f) { return static_cast<la::Fault>(f); }

// Exception -> status code, matching la_status in include/la_cuda.h.
int status_of(const std::exception_ptr& ep, int64_t* bg, int64_t* bp) {
  try {
    std::rethrow_exception(ep);
  } catch (const la::DegenerateDenominator& e) {
    if (bg) *bg = e.group();
    if (bp) *bp = e.position();
    return 6;
  } catch (const la::InvalidShape&) {
    return 1;
  } catch (const la::ShapeMismatch&) {
    return 2;
  } catch (const la::InvalidArgument&) {
    return 3;
  } catch (const la::InvalidPlan&) {
    return 4;
  } catch (const la::MissingForwardState&) {
    return 5;
  } catch (...) {
    return 99;
  }
}

la::HeadTensor wrap(const double* p, int64_t g, int64_t n, int64_t d, int layout) {
  std::vector<double> data(p, p + static_cast<size_t>(g * n * d));
  return la::tensor_from_data({1, g, n, d}, lay(layout), std::move(data));
}

la::BlockPlan plan_of(int64_t g, int64_t n, int64_t d, int64_t l, int workers) {
  la::BlockPlan plan = la::default_plan({1, g, n, d}, workers);
  if (l > 0) plan.reduction_blocks = l;
  return plan;
}

void copy_out(const la::HeadTensor& t, double* dst) {
  std::memcpy(dst, t.flat().data(), sizeof(double) * t.flat().size());
}

}  // namespace

extern "C" {

void ref_make_tensor(double* out, int64_t groups, int64_t n, int64_t d, int layout,
                     uint64_t seed) {
  const la::HeadTensor t =
      la::make_tensor({1, groups, n, d}, lay(layout), la::FillSpec::seeded_uniform(seed));
  copy_out(t, out);
}

// la::forward_causal / la::forward_full (forward.cpp:133-142). out FeatureMajor.
int ref_forward_f64(int causal, const double* q, int lq, const double* k, int lk, const double* v,
                    int lv, int64_t g, int64_t n, int64_t d, double a, double b, int fault,
                    int64_t l, int workers, double* out, double* gvec, int64_t* bg, int64_t* bp) {
  try {
    const auto qt = wrap(q, g, n, d, lq), kt = wrap(k, g, n, d, lk), vt = wrap(v, g, n, d, lv);
    const la::BlockPlan plan = plan_of(g, n, d, l, workers);
    const la::ForwardArtifacts art =
        causal ? la::forward_causal(qt, kt, vt, {a, b}, plan, fault_of(fault))
               : la::forward_full(qt, kt, vt, {a, b}, plan, fault_of(fault));
    copy_out(art.out, out);
    std::memcpy(gvec, art.g.data(), sizeof(double) * art.g.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), bg, bp);
  }
}

// la::backward_causal / la::backward_full (backward.cpp:93-101).
int ref_backward_f64(int causal, const double* q, int lq, const double* k, int lk,
                     const double* v, int lv, const double* o, const double* omega, int lw,
                     const double* gvec, int64_t g, int64_t n, int64_t d, double a, double b,
                     int fault, int64_t l, int workers, double* dq, double* dk, double* dv) {
  try {
    la::ForwardArtifacts art;
    art.q = wrap(q, g, n, d, lq);
    art.k = wrap(k, g, n, d, lk);
    art.v = wrap(v, g, n, d, lv);
    art.out = wrap(o, g, n, d, 0);
    art.g.assign(gvec, gvec + g * n);
    const auto wt = wrap(omega, g, n, d, lw);
    const la::BlockPlan plan = plan_of(g, n, d, l, workers);
    const la::Gradients gr =
        causal ? la::backward_causal(art, wt, {a, b}, plan, fault_of(fault))
               : la::backward_full(art, wt, {a, b}, plan, fault_of(fault));
    copy_out(gr.dq, dq);
    copy_out(gr.dk, dk);
    copy_out(gr.dv, dv);
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// la::quadratic_la (reference.cpp:67-106). out SequenceMajor.
int ref_quadratic(int causal, const double* q, int lq, const double* k, int lk, const double* v,
                  int lv, int64_t g, int64_t n, int64_t d, double a, double b, double* out,
                  double* gvec) {
  try {
    const la::QuadraticResult r =
        la::quadratic_la(wrap(q, g, n, d, lq), wrap(k, g, n, d, lk), wrap(v, g, n, d, lv), {a, b},
                         causal ? la::AttentionMask::Causal : la::AttentionMask::None);
    copy_out(r.out, out);
    std::memcpy(gvec, r.g.data(), sizeof(double) * r.g.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// la::finite_diff_grads (reference.cpp:188-240). Outputs in the input layouts.
int ref_finite_diff(int causal, const double* q, int lq, const double* k, int lk,
                    const double* v, int lv, const double* omega, int lw, int64_t g, int64_t n,
                    int64_t d, double a, double b, double h, double* dq, double* dk, double* dv) {
  try {
    const la::Gradients gr = la::finite_diff_grads(
        wrap(q, g, n, d, lq), wrap(k, g, n, d, lk), wrap(v, g, n, d, lv),
        wrap(omega, g, n, d, lw), {a, b},
        causal ? la::AttentionMask::Causal : la::AttentionMask::None, h);
    copy_out(gr.dq, dq);
    copy_out(gr.dk, dk);
    copy_out(gr.dv, dv);
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// The reference's timed fast path at T=float over raw views (bench.cpp:111-191):
// q,k SequenceMajor; v, omega FeatureMajor; out/dk/dv FeatureMajor; dq SequenceMajor.
int ref_run_forward_f32(int causal, const float* q, const float* k, const float* v, int64_t g,
                        int64_t n, int64_t d, double a, double b, int workers, float* out,
                        float* gvec) {
  try {
    const la::BlockPlan plan = plan_of(g, n, d, 0, workers);
    const auto qv = la::detail::make_const_view(q, g, n, d, la::Layout::SequenceMajor);
    const auto kv = la::detail::make_const_view(k, g, n, d, la::Layout::SequenceMajor);
    const auto vv = la::detail::make_const_view(v, g, n, d, la::Layout::FeatureMajor);
    const auto ov = la::detail::make_mut_view(out, g, n, d, la::Layout::FeatureMajor);
    la::detail::run_forward<float>(qv, kv, vv, {a, b}, plan, causal != 0, la::Fault::None, ov,
                                   gvec);
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

int ref_run_backward_f32(int causal, const float* q, const float* k, const float* v,
                         const float* o, const float* omega, const float* gvec, int64_t g,
                         int64_t n, int64_t d, double a, double b, int workers, float* dq,
                         float* dk, float* dv) {
  try {
    const la::BlockPlan plan = plan_of(g, n, d, 0, workers);
    using la::Layout;
    const auto qv = la::detail::make_const_view(q, g, n, d, Layout::SequenceMajor);
    const auto kv = la::detail::make_const_view(k, g, n, d, Layout::SequenceMajor);
    const auto vv = la::detail::make_const_view(v, g, n, d, Layout::FeatureMajor);
    const auto ov = la::detail::make_const_view(o, g, n, d, Layout::FeatureMajor);
    const auto wv = la::detail::make_const_view(omega, g, n, d, Layout::FeatureMajor);
    const auto dqv = la::detail::make_mut_view(dq, g, n, d, Layout::SequenceMajor);
    const auto dkv = la::detail::make_mut_view(dk, g, n, d, Layout::FeatureMajor);
    const auto dvv = la::detail::make_mut_view(dv, g, n, d, Layout::FeatureMajor);
    la::detail::run_backward<float>(qv, kv, vv, ov, wv, gvec, {a, b}, plan, causal != 0,
                                    la::Fault::None, dqv, dkv, dvv);
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// Term passes (forward.cpp:97-131, backward.cpp:103-153) on a FeatureMajor f64
// accumulator `acc` (in/out, G*N*D). kind 0 constant(v=x), 1 linear(q, k=y, v=z),
// 2 alpha(q, v=y, omega_hat=z), 3 beta(q, o=y, omega_hat=z). Inputs SequenceMajor
// or FeatureMajor per their layout codes.
int ref_term_pass(int kind, const double* x, int lx, const double* y, int ly, const double* z, int lz,
                  int64_t g, int64_t n, int64_t d, double a, double b, int64_t l, double* acc) {
  try {
    la::TermAccumulator f = la::make_accumulator(g, n, d);
    std::memcpy(f.data.data(), acc, sizeof(double) * f.data.size());
    const la::BlockPlan plan = plan_of(g, n, d, l, 2);
    if (kind == 0) {
      la::constant_term_pass(wrap(x, g, n, d, lx), {a, b}, f);
    } else if (kind == 1) {
      la::linear_term_pass(wrap(x, g, n, d, lx), wrap(y, g, n, d, ly), wrap(z, g, n, d, lz), {a, b}, plan, f);
    } else if (kind == 2) {
      la::alpha_term_pass(wrap(x, g, n, d, lx), wrap(y, g, n, d, ly), wrap(z, g, n, d, lz), plan, f, b);
    } else {
      la::beta_term_pass(wrap(x, g, n, d, lx), wrap(y, g, n, d, ly), wrap(z, g, n, d, lz), plan, f, b);
    }
    std::memcpy(acc, f.data.data(), sizeof(double) * f.data.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// la::make_omega_hat (backward.cpp:74-91): out FeatureMajor.
int ref_make_omega_hat(const double* w, int lw, const double* gvec, int64_t g, int64_t n, int64_t d,
                       double* out) {
  try {
    const std::vector<double> gv(gvec, gvec + g * n);
    copy_out(la::make_omega_hat(wrap(w, g, n, d, lw), gv), out);
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// la::normalize_qk (plan.cpp:95-117): both outputs keep their input layouts.
int ref_normalize_qk(const double* q, int lq, const double* k, int lk, int64_t g, int64_t n, int64_t d,
                     double* qo, double* ko) {
  try {
    const auto [a, b] = la::normalize_qk(wrap(q, g, n, d, lq), wrap(k, g, n, d, lk));
    copy_out(a, qo);
    copy_out(b, ko);
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// la::make_prefix_state + la::prefix_advance over `rows` rows (forward.cpp:50-83).
// state = [x1 (d) | x2 (d*d) | y1 | y2 (d)].
int ref_prefix_advance(const double* k_rows, const double* v_rows, int64_t rows, int64_t d, double a,
                       double b, double* state) {
  try {
    la::PrefixState s = la::make_prefix_state(d);
    for (int64_t r = 0; r < rows; ++r)
      s = la::prefix_advance(s, std::span<const double>(k_rows + r * d, d),
                             std::span<const double>(v_rows + r * d, d), {a, b});
    std::memcpy(state, s.x1.data(), sizeof(double) * d);
    std::memcpy(state + d, s.x2.data(), sizeof(double) * d * d);
    state[d + d * d] = s.y1;
    std::memcpy(state + d + d * d + 1, s.y2.data(), sizeof(double) * d);
    return 0;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

// la::read_csv_file + la::fit_slope (bench.cpp:365-403, 459-503): parses a CSV in the
// reference schema and fits log(wall_time_s) against log(N) (axis 0) or log(D) (axis 1)
// over the records with the given pass ("fwd"/"bwd", or "" for all).
int ref_csv_fit(const char* path, int axis, const char* pass, int64_t* n_records, double* slope,
                double* intercept, double* r2) {
  try {
    std::vector<la::BenchRecord> recs = la::read_csv_file(path);
    *n_records = static_cast<int64_t>(recs.size());
    std::vector<la::BenchRecord> sel;
    for (const auto& r : recs)
      if (!pass[0] || std::string(la::pass_name(r.pass)) == pass) sel.push_back(r);
    const la::SlopeFit f = la::fit_slope(sel, axis == 0 ? la::SweepAxis::N : la::SweepAxis::D);
    *slope = f.slope;
    *intercept = f.intercept;
    *r2 = f.r2;
    return 0;
  } catch (const la::IoError&) {
    return 10;
  } catch (const la::InsufficientData&) {
    return 11;
  } catch (...) {
    return status_of(std::current_exception(), nullptr, nullptr);
  }
}

const char* ref_csv_header() { return la::kCsvHeader; }

}  // extern "C"
