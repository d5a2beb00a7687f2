"""Small causal + non-causal fwd/bwd through the public API, for compute-sanitizer runs:
compute-sanitizer --tool racecheck --kernel-regex kns=_tc python tools/sanitize_run.py"""
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
torch.cuda.synchronize()
print("ok")
