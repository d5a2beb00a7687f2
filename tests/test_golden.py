"""Golden fixtures produced by the reference library itself (tests/golden/make_golden.py:
la::forward_* / la::backward_* in f64 on seeded make_tensor inputs), so parity does not
depend on oracle/_ref being present where the tests run.
CPU: the C restatement reproduces them exactly. GPU: the device path (fp32) within 1e-5
relative, Fault mutations included."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import CASES, inputs

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_cases.npz"))
KEYS = ("out", "g", "dq", "dk", "dv")


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_restatement_reproduces_reference_goldens(case):
    name, G, N, D, causal, a, b, seed, fault = case
    q, k, v, w = inputs(G, N, D, seed)
    o, g = O.forward(q, k, v, a, b, causal=causal, fault=fault)
    dq, dk, dv = O.backward(q, k, v, o, w, g, a, b, causal=causal, fault=fault)
    for key, val in zip(KEYS, (o, g, dq, dk, dv)):
        ref = GOLD[f"{name}/{key}"]
        assert np.max(np.abs(val - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref))), (name, key)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_device_fp32_matches_reference_goldens(cuda, case):
    import torch
    import paper_2510_21956_b200 as la
    name, G, N, D, causal, a, b, seed, fault = case
    q, k, v, w = inputs(G, N, D, seed)
    T = lambda x, lay: la.HeadTensor.from_logical(torch.as_tensor(x, dtype=torch.float32).to(cuda), lay)
    L = la.Layout
    c = la.LinearKernelCoeffs(a, b)
    fwd, bwd = (la.forward_causal, la.backward_causal) if causal else (la.forward_full, la.backward_full)
    art = fwd(T(q, L.SequenceMajor), T(k, L.SequenceMajor), T(v, L.FeatureMajor), c, None, la.Fault(fault))
    gr = bwd(art, T(w, L.FeatureMajor), c, None, la.Fault(fault))
    torch.cuda.synchronize()
    got = (art.out.logical(), art.g.cpu().numpy().reshape(G, N), gr.dq.logical(), gr.dk.logical(), gr.dv.logical())
    for key, val in zip(KEYS, got):
        ref = GOLD[f"{name}/{key}"]
        assert np.max(np.abs(val - ref)) / max(np.max(np.abs(ref)), 1e-30) <= 1e-5, (name, key)
