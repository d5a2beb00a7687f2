"""Input prologue and diagnostic entry points: normalize_qk,
relayout, make_omega_hat, the four term passes, prefix_advance.

CPU: the numpy restatements in oracle/oracle.py are pinned against the reference
library itself (oracle/_ref), and the C-ABI validates arguments synchronously with
the reference's exception types. GPU: the device entry points against the
restatements (fp32 <= 1e-5 relative, bf16 <= 2e-2 max-abs on the rounded inputs)."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

FM, SM = O.FEATURE_MAJOR, O.SEQUENCE_MAJOR

needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="reference library not built")


def _inputs(G, N, D, seed):
    rng = np.random.default_rng(seed)
    q, k, v, w, o = (rng.uniform(-1, 1, (G, N, D)) for _ in range(5))
    return O.normalize_rows(q), O.normalize_rows(k), v, w, o


# ----------------------------------------------------------------------------- oracle pinning (CPU)
@needs_ref
@pytest.mark.parametrize("G,N,D,L", [(1, 1, 1, 1), (2, 9, 4, 2), (3, 40, 8, 4), (1, 17, 12, 3)])
def test_term_pass_restatements_match_reference(G, N, D, L):
    q, k, v, w, o = _inputs(G, N, D, G * 100 + N)
    a, b = 0.7, 1.3
    f0 = O.ref_term_pass(0, v, None, None, a, b, np.zeros((G, N, D)), lx=FM, L=L)
    assert np.max(np.abs(f0 - O.constant_term(v, a))) <= 1e-12
    f1 = O.ref_term_pass(1, q, k, v, a, b, f0, lx=SM, ly=SM, lz=FM, L=L)
    assert np.max(np.abs(f1 - O.linear_term(q, k, v, b, f0))) <= 1e-12
    dk = O.ref_term_pass(2, q, v, w, a, b, np.zeros((G, N, D)), lx=SM, ly=FM, lz=FM, L=L)
    assert np.max(np.abs(dk - O.alpha_term(q, v, w, b))) <= 1e-12
    dk2 = O.ref_term_pass(3, q, o, w, a, b, dk, lx=SM, ly=FM, lz=FM, L=L)
    assert np.max(np.abs(dk2 - O.beta_term(q, o, w, b, dk))) <= 1e-12


@needs_ref
def test_term_passes_compose_to_the_forward_numerator():
    # constant + linear = out * g (forward.hpp:53-58); alpha - beta = dK of the forward at unit g
    q, k, v, w, _ = _inputs(2, 24, 6, 5)
    out, g = O.forward(q, k, v, 1.0, 1.0)
    f = O.linear_term(q, k, v, 1.0, O.constant_term(v, 1.0))
    assert np.max(np.abs(f - out * g[:, :, None])) <= 1e-12


@needs_ref
def test_omega_hat_normalize_prefix_match_reference():
    q, k, v, w, _ = _inputs(2, 11, 5, 9)
    g = np.random.default_rng(1).uniform(0.5, 2.0, (2, 11))
    for lw in (FM, SM):
        assert np.array_equal(O.ref_omega_hat(w, g, lw), O.omega_hat(w, g))
    raw = np.random.default_rng(2).uniform(-1, 1, (2, 11, 5))
    raw[0, 3] = 0.0  # zero rows stay zero
    for lq, lk in ((SM, FM), (FM, SM)):
        rq, rk = O.ref_normalize_qk(raw, raw * 2, lq, lk)
        assert np.max(np.abs(rq - O.normalize_rows(raw))) <= 1e-15
        assert np.max(np.abs(rk - O.normalize_rows(raw * 2))) <= 1e-15
        assert np.all(rq[0, 3] == 0.0)
    import paper_2510_21956_b200 as la
    st = la.make_prefix_state(5)
    for r in range(6):
        st = la.prefix_advance(st, k[0, r], v[0, r], la.LinearKernelCoeffs(0.5, 1.5))
    x1, x2, y1, y2 = O.ref_prefix_advance(k[0, :6], v[0, :6], 0.5, 1.5)
    assert np.array_equal(st.x1, x1) and np.array_equal(st.x2, x2) and st.y1 == y1 and np.array_equal(st.y2, y2)


# ----------------------------------------------------------------------------- C-ABI validation (CPU)
def test_prologue_abi_rejects_bad_arguments_synchronously():
    from paper_2510_21956_b200 import _abi
    L = _abi.lib()
    err = _abi.ErrorInfo()
    p = _abi.make_problem(0, 8, 4, "f32")
    assert L.la_normalize_qk(C.byref(p), 1, 1, 1, 1, 1, 1, None, C.byref(err)) == 1  # InvalidShape
    p = _abi.make_problem(1, 8, 4, "f32")
    assert L.la_make_omega_hat(C.byref(p), 1, 0, None, 1, None, C.byref(err)) == 5  # MissingForwardState
    p = _abi.make_problem(1, 8, 4, "f32", a=0.0, b=0.0)
    assert L.la_linear_term_pass(C.byref(p), 1, 1, 1, 1, 1, 0, 1, None, C.byref(err)) == 3  # InvalidArgument
    p = _abi.make_problem(1, 8, 4, "f32")
    p.plan.reduction_blocks = 3  # L must divide D
    assert L.la_alpha_term_pass(C.byref(p), 1, 1, 1, 0, 1, 0, 1, None, C.byref(err)) == 4  # InvalidPlan
    assert b"divide" in err.message or err.message


# ----------------------------------------------------------------------------- device parity (GPU)
def _dev(x, layout, dtype, cuda):
    import torch
    import paper_2510_21956_b200 as la
    t = torch.as_tensor(np.asarray(x, np.float64)).to(getattr(torch, {"f32": "float32", "bf16": "bfloat16"}[dtype]))
    rounded = t.double().numpy()
    return la.HeadTensor.from_logical(t.to(cuda), layout), rounded


def _close(dev, ref, dtype):
    if dtype == "f32":
        return np.max(np.abs(dev - ref)) / max(np.max(np.abs(ref)), 1e-30) <= 1e-5
    return np.max(np.abs(dev - ref)) <= 2e-2


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("G,N,D", [(1, 1, 8), (2, 37, 64), (3, 300, 128), (1, 70, 256)])
def test_term_passes_on_device(cuda, dtype, G, N, D):
    import torch
    import paper_2510_21956_b200 as la
    q, k, v, w, o = _inputs(G, N, D, N + D)
    lays = (SM, FM) if N % 2 else (FM, SM)
    hq, q = _dev(q, lays[0], dtype, cuda)
    hk, k = _dev(k, lays[1], dtype, cuda)
    hv, v = _dev(v, lays[1], dtype, cuda)
    hw, w = _dev(w, FM, dtype, cuda)
    ho, o = _dev(o, lays[0], dtype, cuda)
    c = la.LinearKernelCoeffs(0.8, 1.2)
    plan = la.default_plan(la.Shape(1, G, N, D))
    f = la.make_accumulator(G, N, D)
    la.constant_term_pass(hv, c, f)
    torch.cuda.synchronize()
    f_ref = O.constant_term(v, c.a)
    assert _close(f.logical(), f_ref, "f32")
    la.linear_term_pass(hq, hk, hv, c, plan, f)
    assert _close(f.logical(), O.linear_term(q, k, v, c.b, f_ref), dtype)
    dk = la.make_accumulator(G, N, D)
    la.alpha_term_pass(hq, hv, hw, plan, dk, c.b)
    a_ref = O.alpha_term(q, v, w, c.b)
    assert _close(dk.logical(), a_ref, dtype)
    la.beta_term_pass(hq, ho, hw, plan, dk, c.b)
    assert _close(dk.logical(), O.beta_term(q, o, w, c.b, a_ref), dtype)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("G,N,D", [(1, 1, 3), (2, 33, 64), (2, 257, 128), (1, 65, 256)])
def test_normalize_relayout_omega_hat_on_device(cuda, dtype, G, N, D):
    import torch
    import paper_2510_21956_b200 as la
    rng = np.random.default_rng(G + N + D)
    raw = rng.uniform(-1, 1, (G, N, D))
    raw[0, 0] = 0.0
    for lay in (SM, FM):
        hx, x = _dev(raw, lay, dtype, cuda)
        hq, hk = la.normalize_qk(hx, hx)
        torch.cuda.synchronize()
        assert hq.layout() == lay
        ref = O.normalize_rows(x)
        assert np.max(np.abs(hq.logical() - ref)) <= (1e-6 if dtype == "f32" else 8e-3)
        assert np.all(hq.logical()[0, 0] == 0.0)
        other = FM if lay == SM else SM
        r = la.relayout(hx, other)
        assert r.layout() == other and np.array_equal(r.logical(), x)  # exact copy
        g = rng.uniform(0.5, 3.0, (G, N))
        wh = la.make_omega_hat(hx, torch.as_tensor(g.reshape(-1), dtype=torch.float32, device=cuda))
        assert wh.layout() == la.Layout.FeatureMajor
        ref = O.omega_hat(x, g.astype(np.float32))
        assert np.max(np.abs(wh.logical() - ref)) <= (1e-6 if dtype == "f32" else 8e-3)
