"""Generic 16-bit tensor-core path (csrc/la_g16.cu) against the f64 oracle: head
dimensions the specialised kernels do not take (causal D != 128, up to 256), any
layout of q, k, v, omega, and the three Fault mutations (fault.hpp:7-15), bf16 and
fp16, forced onto the tensor core (impl="tcgen05": no CUDA-core fallback).
Bar: 2e-2 max-abs (BASELINE.json, bf16 against an fp32/f64 oracle)."""
import numpy as np
import pytest

import paper_2510_21956_b200 as la
from tests._util import FM, SM, fast_inputs, max_abs
from tests.test_parity_gpu import oracle_all, run_dev

pytestmark = pytest.mark.gpu

BF16_ABS = 2e-2


def _check(res, causal, a=1.0, b=1.0, fault=0):
    ref = oracle_all(res, causal, a, b, fault=fault)
    errs = {k: max_abs(res[k], ref[k]) for k in ("out", "dq", "dk", "dv") if k in res}
    gerr = float(np.max(np.abs(res["g"] - ref["g"]) / np.abs(ref["g"])))
    assert all(e <= BF16_ABS for e in errs.values()) and gerr <= 1e-3, (errs, gerr)
    return errs


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("D", [32, 64, 96, 192, 256])
def test_generic_head_dims(cuda, dtype, causal, D):
    q, k, v, w = fast_inputs(2, 2048, D, seed=D)
    res = run_dev(q, k, v, w, dtype, cuda, causal=causal, impl="tcgen05")
    _check(res, causal)


@pytest.mark.parametrize("lq,lk,lv,lw", [(FM, FM, SM, SM), (SM, FM, FM, SM), (FM, SM, SM, FM)])
@pytest.mark.parametrize("D", [64, 128])
def test_generic_layouts(cuda, lq, lk, lv, lw, D):
    q, k, v, w = fast_inputs(3, 1024, D, seed=7)
    for causal in (True, False):
        res = run_dev(q, k, v, w, "bf16", cuda, causal=causal, impl="tcgen05", lq=lq, lk=lk, lv=lv, lw=lw)
        _check(res, causal)


@pytest.mark.parametrize("fault", [1, 2, 3])
@pytest.mark.parametrize("causal", [True, False])
def test_generic_faults(cuda, fault, causal):
    # the mutation gate (acceptance.cpp:193-217) on the tensor core: each Fault matches the
    # oracle run with the same Fault, and differs from the clean run
    q, k, v, w = fast_inputs(2, 1024, 128, seed=fault)
    res = run_dev(q, k, v, w, "bf16", cuda, causal=causal, impl="tcgen05", fault=la.Fault(fault))
    _check(res, causal, fault=fault)
    if causal or fault != 2:  # the prefix fault is a no-op without the causal mask
        clean = run_dev(q, k, v, w, "bf16", cuda, causal=causal, impl="tcgen05")
        assert max(max_abs(res[k_], clean[k_]) for k_ in ("out", "dq", "dk", "dv")) > 5e-4


def test_generic_multi_segment_carries(cuda):
    # small G: many segments per group (aggregate units + scanned carries, both directions)
    q, k, v, w = fast_inputs(1, 8192, 64, seed=3)
    for causal in (True, False):
        res = run_dev(q, k, v, w, "bf16", cuda, causal=causal, impl="tcgen05")
        _check(res, causal)
