"""Small causal + non-causal fwd/bwd through the public API, for compute-sanitizer runs:
compute-sanitizer --tool racecheck --kernel-regex kns=_tc python tools/sanitize_run.py
(also exercises the prologue / term-pass kernels)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_21956_b200 as la  # noqa: E402
from tests._util import fast_inputs  # noqa: E402

q, k, v, w = fast_inputs(2, 1024, 128, seed=3)
for causal in (True, False):
    def T(x, lay):
        return la.HeadTensor.from_logical(torch.as_tensor(x).bfloat16().cuda(), lay)
    hq, hk = T(q, la.Layout.SequenceMajor), T(k, la.Layout.SequenceMajor)
    hv, hw = T(v, la.Layout.FeatureMajor), T(w, la.Layout.FeatureMajor)
    art = (la.forward_causal if causal else la.forward_full)(hq, hk, hv)
    (la.backward_causal if causal else la.backward_full)(art, hw)
# prologue / diagnostics kernels (la_prologue.cu)
hq2, hk2 = la.normalize_qk(hq, hk)
hw_hat = la.make_omega_hat(hw, art.g)
la.relayout(hv, la.Layout.SequenceMajor)
plan = la.default_plan(la.Shape(1, 2, 1024, 128))
f = la.make_accumulator(2, 1024, 128)
la.constant_term_pass(hv, la.LinearKernelCoeffs(), f)
la.linear_term_pass(hq, hk, hv, la.LinearKernelCoeffs(), plan, f)
dk = la.make_accumulator(2, 1024, 128)
la.alpha_term_pass(hq, hv, hw_hat, plan, dk)
la.beta_term_pass(hq, art.out, hw_hat, plan, dk)
torch.cuda.synchronize()
print("ok")
