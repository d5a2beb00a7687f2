"""fp32 inputs on the tensor core (csrc/la_f32tc.cu, 3xTF32) against the f64 oracle.

The bar is BASELINE.json's fp32 tolerance, <= 1e-5 relative (max|x-y|/max|y|), for the
forward (out, g) and all three gradients, causal and non-causal, with the kernel forced
(impl="tcgen05": a shape the path does not take fails instead of falling back)."""
import numpy as np
import pytest

import paper_2510_21956_b200 as la
from oracle import oracle as O
from tests._util import bench_inputs, fast_inputs, rel_err
from tests.test_parity_gpu import oracle_all, run_dev

pytestmark = pytest.mark.gpu

FP32_REL = 1e-5


def _check(res, causal, a=1.0, b=1.0, keys=("out", "g", "dq", "dk", "dv")):
    ref = oracle_all(res, causal, a, b)
    errs = {k: rel_err(res[k], ref[k]) for k in keys if k in res}
    assert all(e <= FP32_REL for e in errs.values()), errs
    return errs


@pytest.mark.parametrize("causal", [True, False])
def test_config1_fp32_on_tensor_core(cuda, causal):
    # BASELINE config 1: fp32 B=1 H=4 N=2048 D=64 a=b=1, reference inputs (bench.cpp:75-97)
    q, k, v, w = bench_inputs(4, 2048, 64)
    res = run_dev(q, k, v, w, "f32", cuda, causal=causal, impl="tcgen05")
    _check(res, causal)


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("G,N,D", [(2, 4096, 128), (3, 1024, 32), (1, 640, 100), (5, 128, 64)])
def test_fp32_tc_shapes(cuda, causal, G, N, D):
    # multi-segment carries (G * P ~ one wave), zero-padded feature tiles (D < 128)
    q, k, v, w = fast_inputs(G, N, D, seed=G + N + D)
    res = run_dev(q, k, v, w, "f32", cuda, causal=causal, impl="tcgen05")
    _check(res, causal)


@pytest.mark.parametrize("a,b", [(0.5, 2.0), (1.0, 0.0), (2.0, -0.25)])
def test_fp32_tc_coefficients(cuda, a, b):
    q, k, v, w = fast_inputs(2, 1024, 64, seed=31)
    for causal in (True, False):
        res = run_dev(q, k, v, w, "f32", cuda, causal=causal, a=a, b=b, impl="tcgen05")
        _check(res, causal, a, b)


def test_fp32_tc_matches_cuda_core_path(cuda):
    q, k, v, w = fast_inputs(2, 2048, 128, seed=5)
    tc = run_dev(q, k, v, w, "f32", cuda, impl="tcgen05")
    si = run_dev(q, k, v, w, "f32", cuda, impl="simt")
    for key in ("out", "g", "dq", "dk", "dv"):
        assert rel_err(tc[key], si[key]) <= FP32_REL, key


def test_fp32_tc_degenerate_denominator(cuda):
    # g_1 = 2a + b q_1 . (k_0 + k_1) = 0 with q_1 = -e0, k = e0: DegenerateDenominator(0, 1)
    N, D = 64, 8
    q = np.zeros((1, N, D))
    q[0, :, 0] = 1.0
    q[0, 1, 0] = -1.0
    k = np.zeros((1, N, D))
    k[0, :, 0] = 1.0
    v = O.seeded(1, N, D, 90, O.FEATURE_MAJOR)
    with pytest.raises(la.DegenerateDenominator) as e:
        run_dev(q, k, v, None, "f32", cuda, impl="tcgen05")
    assert (e.value.group(), e.value.position()) == (0, 1)


@pytest.mark.parametrize("fault", [1, 2, 3])
@pytest.mark.parametrize("causal", [True, False])
def test_fp32_tc_faults(cuda, fault, causal):
    # the Fault mutations (fault.hpp:7-15) on the tensor core match the oracle with the same fault
    q, k, v, w = bench_inputs(2, 512, 32, seed=fault)
    res = run_dev(q, k, v, w, "f32", cuda, causal=causal, impl="tcgen05", fault=la.Fault(fault))
    ref = oracle_all(res, causal, fault=fault)
    for key in ("out", "g", "dq", "dk", "dv"):
        assert rel_err(res[key], ref[key]) <= FP32_REL, key


def test_fp32_tc_mixed_layouts(cuda):
    from tests._util import FM, SM
    q, k, v, w = fast_inputs(2, 1024, 64, seed=12)
    for causal in (True, False):
        res = run_dev(q, k, v, w, "f32", cuda, causal=causal, impl="tcgen05", lq=FM, lk=FM, lv=SM, lw=SM)
        _check(res, causal)
