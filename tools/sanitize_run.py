"""Small causal + non-causal fwd/bwd through the public API, for compute-sanitizer runs:
compute-sanitizer --tool racecheck --kernel-regex kns=_tc python tools/sanitize_run.py
(also exercises the prologue / term-pass kernels). With --round2 it runs instead the kernels
added in round 2: non-causal D = 64 / 256 (la_full.cu), causal D = 192 and a non-canonical
layout (la_g16.cu), fp32 inputs (la_f32tc.cu), the cluster-pair backward (la_bwd_pair.cu)
and a small-G causal step long enough for the carry scan (k_seg_scan)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_21956_b200 as la  # noqa: E402
from tests._util import fast_inputs  # noqa: E402

from paper_2510_21956_b200 import _abi  # noqa: E402

if "--round2" in sys.argv:
    def H(x, lay, dt=torch.bfloat16):
        return la.HeadTensor.from_logical(torch.as_tensor(x).to(dt).cuda(), lay)
    SM_, FM_ = la.Layout.SequenceMajor, la.Layout.FeatureMajor
    for (G, N, D, causal, dt, lq) in ((2, 1024, 64, False, torch.bfloat16, SM_),
                                      (2, 1024, 256, False, torch.bfloat16, SM_),
                                      (2, 1024, 192, True, torch.bfloat16, SM_),
                                      (2, 1024, 128, True, torch.bfloat16, FM_),
                                      (2, 1024, 64, True, torch.float32, SM_),
                                      (2, 4096, 128, True, torch.bfloat16, SM_)):
        q, k, v, w = fast_inputs(G, N, D, seed=5)
        hq, hk, hv, hw = H(q, lq, dt), H(k, SM_, dt), H(v, FM_, dt), H(w, FM_, dt)
        art = (la.forward_causal if causal else la.forward_full)(hq, hk, hv)
        (la.backward_causal if causal else la.backward_full)(art, hw)
    q, k, v, w = fast_inputs(2, 2048, 128, seed=6)  # the opt-in cluster-pair backward
    art = la.forward_causal(H(q, SM_), H(k, SM_), H(v, FM_))
    _abi.set_tuning(bwd_pair=1)
    la.backward_causal(art, H(w, FM_))
    _abi.set_tuning()
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)

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
