// GPU verify suites through the reference-side shim (la::cuda::*, la_cuda_shim.cpp).
//
// TEST INFRASTRUCTURE: mirrors the reference's `la verify` suites
// (proj/src/verify.cpp:57-380) and the mutation-sensitivity gate
// (proj/tests/acceptance.cpp:193-217), but with the device path as the code under
// test. The checkers are the reference library itself (oracle/_ref/libla_ref.so,
// f64): quadratic_la (reference.cpp:67-106) for the forward, the reference's own
// analytic backward_causal/backward_full for the gradients. Built by oracle/Makefile
// into oracle/_ref/verify_gpu; run on the GPU box by tests/test_integration.py.
//
// Suites (same case generators as verify.cpp: seeded mt19937_64 draws of n, d,
// heads, mask, coefficients and layouts; row-normalised q, k):
//   forward    device forward_* vs quadratic_la            fp32: <= 1e-5 relative
//   backward   device backward_* vs reference backward_*   fp32: <= 1e-5 relative
//   plan       device outputs bitwise identical across L in {1,2,4} x workers {1,4,8}
//   normalize  normalized draws never give g_i <= 0 or DegenerateDenominator on the device
//   faults     (clean runs only) every Fault on the device equals the reference's
//              faulted result, so the injected defects are the reference's defects
//   tensorcore bf16 through the shim: N = 256 / 512 / 300 (padded), D = 128 / 64 causal and
//              non-causal, D = 256 non-causal, vs the f64 reference on the bf16-rounded
//              inputs: <= 2e-2 max-abs
// Exit 0 when every suite passes, 1 otherwise (--inject-defect makes the device run
// the named Fault, which the forward or backward suite must then catch).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "la/backward.hpp"
#include "la/error.hpp"
#include "la/forward.hpp"
#include "la/plan.hpp"
#include "la/reference.hpp"
#include "la/tensor.hpp"

namespace la::cuda {  // integration/la_cuda_shim.cpp
ForwardArtifacts forward_causal(const HeadTensor&, const HeadTensor&, const HeadTensor&,
                                const LinearKernelCoeffs&, const BlockPlan&, Fault);
ForwardArtifacts forward_full(const HeadTensor&, const HeadTensor&, const HeadTensor&,
                              const LinearKernelCoeffs&, const BlockPlan&, Fault);
Gradients backward_causal(const ForwardArtifacts&, const HeadTensor&, const LinearKernelCoeffs&,
                          const BlockPlan&, Fault);
Gradients backward_full(const ForwardArtifacts&, const HeadTensor&, const LinearKernelCoeffs&,
                        const BlockPlan&, Fault);
}  // namespace la::cuda

using namespace la;

namespace {

struct Opts {
  uint64_t seed = 0;
  size_t fwd_cases = 200, bwd_cases = 100, norm_cases = 2000, tc_cases = 7;
  Fault fault = Fault::None;
  bool bf16 = false;
};

struct Result {
  std::string name;
  bool passed = false;
  size_t cases = 0;
  double max_dev = 0.0, tol = 0.0;
  std::string detail;
};

HeadTensor seeded(const Shape& s, Layout l, uint64_t seed) {
  return make_tensor(s, l, FillSpec::seeded_uniform(seed, -1.0, 1.0));
}

// max |x - y| / max |y| over logical elements (layouts may differ)
double rel_dev(const HeadTensor& x, const HeadTensor& y) {
  double num = 0.0, den = 0.0;
  for (int64_t g = 0; g < y.groups(); ++g)
    for (int64_t i = 0; i < y.seq_len(); ++i)
      for (int64_t j = 0; j < y.dim(); ++j) {
        num = std::max(num, std::fabs(x.at(g, i, j) - y.at(g, i, j)));
        den = std::max(den, std::fabs(y.at(g, i, j)));
      }
  return den > 0 ? num / den : num;
}
double abs_dev(const HeadTensor& x, const HeadTensor& y) {
  double num = 0.0;
  for (int64_t g = 0; g < y.groups(); ++g)
    for (int64_t i = 0; i < y.seq_len(); ++i)
      for (int64_t j = 0; j < y.dim(); ++j) num = std::max(num, std::fabs(x.at(g, i, j) - y.at(g, i, j)));
  return num;
}
double max_abs(const HeadTensor& y) {
  double m = 0.0;
  for (double x : y.flat()) m = std::max(m, std::fabs(x));
  return m;
}
double rel_dev(const std::vector<double>& x, const std::vector<double>& y) {
  double num = 0.0, den = 0.0;
  for (size_t e = 0; e < y.size(); ++e) {
    num = std::max(num, std::fabs(x[e] - y[e]));
    den = std::max(den, std::fabs(y[e]));
  }
  return den > 0 ? num / den : num;
}
bool well_conditioned(const std::vector<double>& g) {  // verify.cpp:34-42 floor
  for (double gi : g)
    if (std::fabs(gi) < 0.25) return false;
  return true;
}
bool flat_equal(const HeadTensor& x, const HeadTensor& y) {
  auto a = x.flat(), b = y.flat();
  return a.size() == b.size() && std::equal(a.begin(), a.end(), b.begin());
}
HeadTensor round_bf16(const HeadTensor& t) {  // RNE, the shim's staging rounding
  std::vector<double> d(t.flat().begin(), t.flat().end());
  for (double& x : d) {
    float f = (float)x;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000u;
    std::memcpy(&f, &u, 4);
    x = f;
  }
  return wrap_unchecked(t.groups(), t.seq_len(), t.dim(), t.layout(), std::move(d));
}

ForwardArtifacts dev_fwd(bool causal, const HeadTensor& q, const HeadTensor& k, const HeadTensor& v,
                         const LinearKernelCoeffs& c, const BlockPlan& p, Fault f) {
  return causal ? cuda::forward_causal(q, k, v, c, p, f) : cuda::forward_full(q, k, v, c, p, f);
}
Gradients dev_bwd(bool causal, const ForwardArtifacts& a, const HeadTensor& w, const LinearKernelCoeffs& c,
                  const BlockPlan& p, Fault f) {
  return causal ? cuda::backward_causal(a, w, c, p, f) : cuda::backward_full(a, w, c, p, f);
}
ForwardArtifacts ref_fwd(bool causal, const HeadTensor& q, const HeadTensor& k, const HeadTensor& v,
                         const LinearKernelCoeffs& c, const BlockPlan& p, Fault f) {
  return causal ? la::forward_causal(q, k, v, c, p, f) : la::forward_full(q, k, v, c, p, f);
}
Gradients ref_bwd(bool causal, const ForwardArtifacts& a, const HeadTensor& w, const LinearKernelCoeffs& c,
                  const BlockPlan& p, Fault f) {
  return causal ? la::backward_causal(a, w, c, p, f) : la::backward_full(a, w, c, p, f);
}

Result forward_suite(const Opts& o) {
  Result r{"forward"};
  r.tol = 1e-5;
  const LinearKernelCoeffs coeff[] = {{1.0, 1.0}, {1.0, 0.5}, {0.3, 1.0}};
  std::mt19937_64 rng(o.seed ^ 0xf0f0a1a1u);
  size_t att = 0;
  double gdev = 0.0;
  while (r.cases < o.fwd_cases && att < o.fwd_cases * 4 + 64) {
    ++att;
    const int64_t n = (int64_t)(rng() % 64) + 1, d = (int64_t)(rng() % 32) + 1, h = (int64_t)(rng() % 3) + 1;
    const Shape s{1, h, n, d};
    const bool causal = att % 2 == 0;
    const LinearKernelCoeffs c = coeff[att % 3];
    const Layout lq = rng() % 2 ? Layout::SequenceMajor : Layout::FeatureMajor;
    const Layout lk = rng() % 2 ? Layout::SequenceMajor : Layout::FeatureMajor;
    const Layout lv = rng() % 2 ? Layout::SequenceMajor : Layout::FeatureMajor;
    const auto [q, k] = normalize_qk(seeded(s, lq, rng()), seeded(s, lk, rng()));
    const HeadTensor v = seeded(s, lv, rng());
    QuadraticResult ora;
    try {
      ora = quadratic_la(q, k, v, c, causal ? AttentionMask::Causal : AttentionMask::None);
    } catch (const DegenerateDenominator&) {
      continue;
    }
    if (!well_conditioned(ora.g)) continue;
    ForwardArtifacts dev;
    try {
      dev = dev_fwd(causal, q, k, v, c, default_plan(s, 1), o.fault);
    } catch (const DegenerateDenominator&) {
      continue;
    }
    r.max_dev = std::max(r.max_dev, rel_dev(dev.out, ora.out));
    gdev = std::max(gdev, rel_dev(dev.g, ora.g));
    ++r.cases;
  }
  r.passed = r.cases >= o.fwd_cases && r.max_dev <= r.tol && gdev <= r.tol;
  char b[160];
  std::snprintf(b, sizeof b, "max rel |device - quadratic| out %.3e, g %.3e", r.max_dev, gdev);
  r.detail = b;
  return r;
}

Result backward_suite(const Opts& o) {
  Result r{"backward"};
  r.tol = 1e-5;
  const LinearKernelCoeffs coeff[] = {{1.0, 1.0}, {1.0, 0.3}};
  std::mt19937_64 rng(o.seed ^ 0xbdbd0202u);
  size_t att = 0;
  while (r.cases < o.bwd_cases && att < o.bwd_cases * 4 + 64) {
    ++att;
    const int64_t n = (int64_t)(rng() % 32) + 1, d = (int64_t)(rng() % 8) + 1, h = (int64_t)(rng() % 2) + 1;
    const Shape s{1, h, n, d};
    const bool causal = att % 2 == 0;
    const LinearKernelCoeffs c = coeff[att % 2];
    const auto [q, k] = normalize_qk(seeded(s, Layout::SequenceMajor, rng()),
                                     seeded(s, Layout::SequenceMajor, rng()));
    const HeadTensor v = seeded(s, Layout::FeatureMajor, rng());
    const HeadTensor w = seeded(s, Layout::FeatureMajor, rng());
    const BlockPlan plan = default_plan(s, 1);
    try {
      const ForwardArtifacts ra = ref_fwd(causal, q, k, v, c, plan, Fault::None);
      if (!well_conditioned(ra.g)) continue;
      const Gradients rg = ref_bwd(causal, ra, w, c, plan, Fault::None);
      const ForwardArtifacts da = dev_fwd(causal, q, k, v, c, plan, Fault::None);
      const Gradients dg = dev_bwd(causal, da, w, c, plan, o.fault);
      // relative to the case's gradient scale: single-row causal dq is exactly 0 in
      // f64 (the alpha and beta terms cancel), so a per-tensor max|y| can vanish
      const double scale = std::max({max_abs(rg.dq), max_abs(rg.dk), max_abs(rg.dv)});
      const double dev = std::max({abs_dev(dg.dq, rg.dq), abs_dev(dg.dk, rg.dk), abs_dev(dg.dv, rg.dv)});
      r.max_dev = std::max(r.max_dev, scale > 0 ? dev / scale : dev);
    } catch (const DegenerateDenominator&) {
      continue;
    }
    ++r.cases;
  }
  r.passed = r.cases >= o.bwd_cases && r.max_dev <= r.tol;
  char b[160];
  std::snprintf(b, sizeof b, "max |device - reference analytic| over dq, dk, dv / max |reference gradient| %.3e", r.max_dev);
  r.detail = b;
  return r;
}

Result plan_suite(const Opts& o) {  // verify.cpp:243-290
  Result r{"plan"};
  const Shape s{1, 2, 128, 64};
  const LinearKernelCoeffs c{1.0, 1.0};
  const HeadTensor q = seeded(s, Layout::SequenceMajor, o.seed + 11);
  const HeadTensor k = seeded(s, Layout::SequenceMajor, o.seed + 12);
  const HeadTensor v = seeded(s, Layout::FeatureMajor, o.seed + 13);
  const HeadTensor w = seeded(s, Layout::FeatureMajor, o.seed + 14);
  bool same = true;
  for (const bool causal : {true, false}) {
    BlockPlan base = default_plan(s, 1);
    base.reduction_blocks = 1;
    base.workers = 1;
    const ForwardArtifacts ba = dev_fwd(causal, q, k, v, c, base, o.fault);
    const Gradients bg = dev_bwd(causal, ba, w, c, base, o.fault);
    for (const int64_t l : {1, 2, 4})
      for (const int wk : {1, 4, 8}) {
        BlockPlan p = base;
        p.reduction_blocks = l;
        p.workers = wk;
        const ForwardArtifacts a = dev_fwd(causal, q, k, v, c, p, o.fault);
        const Gradients gr = dev_bwd(causal, a, w, c, p, o.fault);
        same = same && flat_equal(a.out, ba.out) && a.g == ba.g && flat_equal(gr.dq, bg.dq) &&
               flat_equal(gr.dk, bg.dk) && flat_equal(gr.dv, bg.dv);
        ++r.cases;
      }
  }
  r.passed = same;
  r.max_dev = same ? 0.0 : 1.0;
  r.detail = same ? "device outputs and gradients bitwise identical across L x workers" : "outputs differ across plans";
  return r;
}

Result normalize_suite(const Opts& o) {  // verify.cpp:345-382
  Result r{"normalize"};
  std::mt19937_64 rng(o.seed ^ 0x5151dedeu);
  const LinearKernelCoeffs c{1.0, 1.0};
  size_t degenerate = 0, nonpos = 0;
  for (size_t i = 0; i < o.norm_cases; ++i) {
    const int64_t n = (int64_t)(rng() % 128) + 1, d = (int64_t)(rng() % 61) + 4;
    const Shape s{1, 1, n, d};
    const HeadTensor qr = seeded(s, Layout::SequenceMajor, rng());
    const HeadTensor kr = seeded(s, Layout::SequenceMajor, rng());
    const HeadTensor v = seeded(s, Layout::FeatureMajor, rng());
    const auto [q, k] = normalize_qk(qr, kr);
    try {
      const ForwardArtifacts a = cuda::forward_causal(q, k, v, c, default_plan(s, 1), o.fault);
      for (double gi : a.g)
        if (!(gi > 0.0)) ++nonpos;
    } catch (const DegenerateDenominator&) {
      ++degenerate;
    }
    ++r.cases;
  }
  r.passed = degenerate == 0 && nonpos == 0;
  r.max_dev = (double)degenerate;
  r.detail = "degenerate denominators: " + std::to_string(degenerate) + ", non-positive g_i: " + std::to_string(nonpos);
  return r;
}

// Each injected defect on the device reproduces the reference's own defect.
Result fault_suite(const Opts& o) {
  Result r{"faults"};
  r.tol = 1e-5;
  std::mt19937_64 rng(o.seed ^ 0xfa17fa17u);
  const LinearKernelCoeffs c{1.0, 0.7};
  for (const Fault f : {Fault::FlipBetaKSign, Fault::CausalPrefixOffByOne, Fault::DropGradVConstantTerm})
    for (const bool causal : {true, false})
      for (int rep = 0; rep < 3; ++rep) {
        const Shape s{1, 2, (int64_t)(rng() % 48) + 8, (int64_t)(rng() % 16) + 4};
        const auto [q, k] = normalize_qk(seeded(s, Layout::SequenceMajor, rng()),
                                         seeded(s, Layout::SequenceMajor, rng()));
        const HeadTensor v = seeded(s, Layout::FeatureMajor, rng());
        const HeadTensor w = seeded(s, Layout::FeatureMajor, rng());
        const BlockPlan p = default_plan(s, 1);
        try {
          const ForwardArtifacts ra = ref_fwd(causal, q, k, v, c, p, f);
          const ForwardArtifacts da = dev_fwd(causal, q, k, v, c, p, f);
          const Gradients rg = ref_bwd(causal, ra, w, c, p, f);
          const Gradients dg = dev_bwd(causal, da, w, c, p, f);
          const double scale = std::max({max_abs(rg.dq), max_abs(rg.dk), max_abs(rg.dv)});
          const double gdev = std::max({abs_dev(dg.dq, rg.dq), abs_dev(dg.dk, rg.dk), abs_dev(dg.dv, rg.dv)});
          r.max_dev = std::max({r.max_dev, rel_dev(da.out, ra.out), rel_dev(da.g, ra.g), scale > 0 ? gdev / scale : gdev});
          ++r.cases;
        } catch (const DegenerateDenominator&) {
        }
      }
  r.passed = r.cases >= 12 && r.max_dev <= r.tol;
  char b[160];
  std::snprintf(b, sizeof b, "max rel |device - reference| with the same Fault injected %.3e", r.max_dev);
  r.detail = b;
  return r;
}

// bf16 tensor-core path (N % 128 == 0, D = 128, canonical layouts) through the same shim.
Result tensorcore_suite(const Opts& o) {
  Result r{"tensorcore"};
  r.tol = 2e-2;
  std::mt19937_64 rng(o.seed ^ 0x7c057c05u);
  const LinearKernelCoeffs c{1.0, 1.0};
  setenv("LA_SHIM_DTYPE", "bf16", 1);
  // tcgen05 (N % 128 == 0, D = 128), the padded-N path, D < 128 (zero-padded D causal,
  // batched GEMMs non-causal) and D = 256 non-causal
  const int64_t shapes[][2] = {{256, 128}, {512, 128}, {300, 128}, {300, 128}, {256, 64}, {256, 64}, {200, 256}};
  for (size_t t = 0; t < o.tc_cases; ++t) {
    const int64_t n = shapes[t % 7][0], d = shapes[t % 7][1];
    const bool causal = d == 256 ? false : t % 2 == 0;
    const Shape s{1, 2, n, d};
    const auto [q0, k0] = normalize_qk(seeded(s, Layout::SequenceMajor, rng()),
                                       seeded(s, Layout::SequenceMajor, rng()));
    const HeadTensor q = round_bf16(q0), k = round_bf16(k0);
    const HeadTensor v = round_bf16(seeded(s, Layout::FeatureMajor, rng()));
    const HeadTensor w = round_bf16(seeded(s, Layout::FeatureMajor, rng()));
    const BlockPlan p = default_plan(s, 1);
    const ForwardArtifacts ra = ref_fwd(causal, q, k, v, c, p, Fault::None);
    const ForwardArtifacts da = dev_fwd(causal, q, k, v, c, p, o.fault);
    const Gradients rg = ref_bwd(causal, ra, w, c, p, Fault::None);
    const Gradients dg = dev_bwd(causal, da, w, c, p, o.fault);
    r.max_dev = std::max({r.max_dev, abs_dev(da.out, ra.out), abs_dev(dg.dq, rg.dq), abs_dev(dg.dk, rg.dk),
                          abs_dev(dg.dv, rg.dv)});
    ++r.cases;
  }
  unsetenv("LA_SHIM_DTYPE");
  r.passed = r.max_dev <= r.tol;
  char b[160];
  std::snprintf(b, sizeof b, "bf16 device vs f64 reference on the rounded inputs: max-abs %.3e", r.max_dev);
  r.detail = b;
  return r;
}

Fault parse_fault(const std::string& s) {  // the CLI's --inject-defect names (acceptance.cpp:202-206)
  if (s == "beta-k-sign") return Fault::FlipBetaKSign;
  if (s == "causal-off-by-one") return Fault::CausalPrefixOffByOne;
  if (s == "drop-v-a-term") return Fault::DropGradVConstantTerm;
  std::fprintf(stderr, "unknown defect %s\n", s.c_str());
  std::exit(2);
}

}  // namespace

int main(int argc, char** argv) {
  Opts o;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i], v = argv[i + 1];
    if (a == "--seed") o.seed = std::strtoull(v.c_str(), nullptr, 10);
    else if (a == "--fwd-cases") o.fwd_cases = std::strtoull(v.c_str(), nullptr, 10);
    else if (a == "--bwd-cases") o.bwd_cases = std::strtoull(v.c_str(), nullptr, 10);
    else if (a == "--norm-cases") o.norm_cases = std::strtoull(v.c_str(), nullptr, 10);
    else if (a == "--tc-cases") o.tc_cases = std::strtoull(v.c_str(), nullptr, 10);
    else if (a == "--inject-defect") o.fault = parse_fault(v);
    else {
      std::fprintf(stderr, "unknown option %s\n", a.c_str());
      return 2;
    }
  }
  std::vector<Result> rs;
  try {
    rs.push_back(forward_suite(o));
    rs.push_back(backward_suite(o));
    rs.push_back(plan_suite(o));
    rs.push_back(normalize_suite(o));
    if (o.fault == Fault::None) rs.push_back(fault_suite(o));
    if (o.tc_cases) rs.push_back(tensorcore_suite(o));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "verify_gpu: %s\n", e.what());
    return 3;
  }
  bool ok = true;
  for (const Result& r : rs) {
    std::printf("{\"suite\": \"%s\", \"passed\": %s, \"cases\": %zu, \"max_dev\": %.6e, \"tolerance\": %.1e, "
                "\"detail\": \"%s\"}\n",
                r.name.c_str(), r.passed ? "true" : "false", r.cases, r.max_dev, r.tol, r.detail.c_str());
    ok = ok && r.passed;
  }
  return ok ? 0 : 1;
}
