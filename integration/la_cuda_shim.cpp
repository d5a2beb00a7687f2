// Drop-in shim a maintainer adds to the reference library (proj/src) to route
// la::forward_causal / forward_full / backward_causal / backward_full to the B200
// C-ABI (include/la_cuda.h). Same signatures, same HeadTensor layouts, same
// exception types. Compiled against the reference headers by
// tests/test_integration.py (g++ -fsyntax-only + link check).
//
// Precision: the reference's public API is f64; the device computes in f32
// (LA_F32, <= 1e-5 relative vs the f64 reference) by default. Set
// LA_SHIM_DTYPE=bf16 for the tensor-core path.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "la/backward.hpp"
#include "la/error.hpp"
#include "la/forward.hpp"
#include "la/plan.hpp"
#include "la/tensor.hpp"
#include "la_cuda.h"

namespace la::cuda {

namespace {

[[noreturn]] void rethrow(const la_error_info& e) {
  const std::string msg = e.message;
  switch (e.code) {
    case LA_ERR_INVALID_SHAPE: throw InvalidShape(msg);
    case LA_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
    case LA_ERR_INVALID_ARGUMENT: throw InvalidArgument(msg);
    case LA_ERR_INVALID_PLAN: throw InvalidPlan(msg);
    case LA_ERR_MISSING_FORWARD_STATE: throw MissingForwardState(msg);
    case LA_ERR_DEGENERATE_DENOMINATOR: throw DegenerateDenominator(e.group, e.position);
    default: throw Error(msg);
  }
}

la_problem problem(const HeadTensor& q, const LinearKernelCoeffs& c, const BlockPlan& plan,
                   bool causal, Fault fault) {
  la_problem p{};
  p.groups = q.groups();
  p.seq_len = q.seq_len();
  p.dim = q.dim();
  const char* dt = std::getenv("LA_SHIM_DTYPE");
  p.dtype = (dt && std::string(dt) == "bf16") ? LA_BF16 : LA_F32;
  p.a = c.a;
  p.b = c.b;
  p.causal = causal ? 1 : 0;
  p.fault = static_cast<la_fault>(fault);
  p.impl = LA_IMPL_AUTO;
  p.plan = {plan.groups, plan.reduction_blocks, plan.lanes, plan.workers, plan.deterministic ? 1 : 0};
  return p;
}

la_layout lay(Layout l) { return l == Layout::FeatureMajor ? LA_FEATURE_MAJOR : LA_SEQUENCE_MAJOR; }

// f64 HeadTensor -> f32 host staging (bf16 staging is done with a round-to-nearest cast).
std::vector<uint16_t> to_bf16(const HeadTensor& t) {
  std::vector<uint16_t> out(t.flat().size());
  for (size_t i = 0; i < out.size(); ++i) {
    float f = static_cast<float>(t.flat()[i]);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFF + ((u >> 16) & 1);
    out[i] = static_cast<uint16_t>(u >> 16);
  }
  return out;
}
std::vector<float> to_f32(const HeadTensor& t) { return {t.flat().begin(), t.flat().end()}; }

double from(const la_problem& p, const void* buf, size_t i) {
  if (p.dtype == LA_F32) return static_cast<const float*>(buf)[i];
  uint32_t u = static_cast<uint32_t>(static_cast<const uint16_t*>(buf)[i]) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

struct Staged {
  std::vector<float> f;
  std::vector<uint16_t> h;
  const void* ptr() const { return f.empty() ? static_cast<const void*>(h.data()) : f.data(); }
};
Staged stage(const la_problem& p, const HeadTensor& t) {
  Staged s;
  if (p.dtype == LA_F32) s.f = to_f32(t); else s.h = to_bf16(t);
  return s;
}

HeadTensor wrap(const la_problem& p, const std::vector<uint8_t>& buf, Layout layout) {
  std::vector<double> data(static_cast<size_t>(p.groups * p.seq_len * p.dim));
  for (size_t i = 0; i < data.size(); ++i) data[i] = from(p, buf.data(), i);
  return wrap_unchecked(p.groups, p.seq_len, p.dim, layout, std::move(data));
}

ForwardArtifacts run_forward(const HeadTensor& q, const HeadTensor& k, const HeadTensor& v,
                             const LinearKernelCoeffs& c, const BlockPlan& plan, bool causal,
                             Fault fault) {
  if (q.empty() || k.empty() || v.empty()) throw InvalidShape("forward requires non-empty Q, K, V");
  if (!q.same_shape(k) || !q.same_shape(v)) throw ShapeMismatch("Q, K, V shapes must agree");
  const la_problem p = problem(q, c, plan, causal, fault);
  const size_t n = static_cast<size_t>(q.size()), eb = p.dtype == LA_F32 ? 4 : 2;
  Staged sq = stage(p, q), sk = stage(p, k), sv = stage(p, v);
  std::vector<uint8_t> out(n * eb);
  std::vector<float> g(static_cast<size_t>(q.groups() * q.seq_len()));
  la_error_info err{};
  if (la_host_forward(&p, sq.ptr(), lay(q.layout()), sk.ptr(), lay(k.layout()), sv.ptr(),
                      lay(v.layout()), out.data(), g.data(), &err) != LA_OK)
    rethrow(err);
  ForwardArtifacts art;
  art.out = wrap(p, out, Layout::FeatureMajor);
  art.g.assign(g.begin(), g.end());
  art.q = q;
  art.k = k;
  art.v = v;
  return art;
}

Gradients run_backward(const ForwardArtifacts& art, const HeadTensor& omega,
                       const LinearKernelCoeffs& c, const BlockPlan& plan, bool causal, Fault fault) {
  if (art.out.empty() || art.q.empty() || art.k.empty() || art.v.empty())
    throw MissingForwardState("backward requires the forward artifacts (Q, K, V, O)");
  if (art.g.size() != static_cast<size_t>(art.out.groups() * art.out.seq_len()))
    throw MissingForwardState("backward requires the retained denominator vector g");
  if (omega.empty() || !omega.same_shape(art.out))
    throw ShapeMismatch("cotangent shape must match the forward output");
  const la_problem p = problem(art.q, c, plan, causal, fault);
  const size_t n = static_cast<size_t>(art.q.size()), eb = p.dtype == LA_F32 ? 4 : 2;
  Staged sq = stage(p, art.q), sk = stage(p, art.k), sv = stage(p, art.v), so = stage(p, art.out),
         sw = stage(p, omega);
  std::vector<float> g(art.g.begin(), art.g.end());
  std::vector<uint8_t> dq(n * eb), dk(n * eb), dv(n * eb);
  la_error_info err{};
  if (la_host_backward(&p, sq.ptr(), lay(art.q.layout()), sk.ptr(), lay(art.k.layout()), sv.ptr(),
                       lay(art.v.layout()), so.ptr(), sw.ptr(), lay(omega.layout()), g.data(),
                       dq.data(), dk.data(), dv.data(), &err) != LA_OK)
    rethrow(err);
  Gradients gr;
  gr.dq = wrap(p, dq, Layout::SequenceMajor);
  gr.dk = wrap(p, dk, Layout::FeatureMajor);
  gr.dv = wrap(p, dv, Layout::FeatureMajor);
  return gr;
}

}  // namespace

ForwardArtifacts forward_causal(const HeadTensor& q, const HeadTensor& k, const HeadTensor& v,
                                const LinearKernelCoeffs& c, const BlockPlan& plan, Fault fault) {
  return run_forward(q, k, v, c, plan, true, fault);
}
ForwardArtifacts forward_full(const HeadTensor& q, const HeadTensor& k, const HeadTensor& v,
                              const LinearKernelCoeffs& c, const BlockPlan& plan, Fault fault) {
  return run_forward(q, k, v, c, plan, false, fault);
}
Gradients backward_causal(const ForwardArtifacts& art, const HeadTensor& omega,
                          const LinearKernelCoeffs& c, const BlockPlan& plan, Fault fault) {
  return run_backward(art, omega, c, plan, true, fault);
}
Gradients backward_full(const ForwardArtifacts& art, const HeadTensor& omega,
                        const LinearKernelCoeffs& c, const BlockPlan& plan, Fault fault) {
  return run_backward(art, omega, c, plan, false, fault);
}

}  // namespace la::cuda
