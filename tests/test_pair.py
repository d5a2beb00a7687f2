"""The cluster-pair causal backward (csrc/la_bwd_pair.cu, opt-in through la_tuning.bwd_pair):
parity against the float64 chunked oracle and agreement with the segmented sweep on the same
inputs, at small sizes and at the north-star launch geometry (one pair sweeps all 65536 rows
of a group, with the forward's segment-end and checkpoint prefixes reloaded on the way).

Bars as tests/test_parity_geometry.py: bf16 <= 2e-2 max-abs and <= 1e-2 relative against the
oracle; the two device paths differ only in fp32 summation order and bf16 rounding of the
state operands, so they agree to a few bf16 ulps (<= 4e-3 max-abs here)."""
import ctypes as C

import pytest

from tests import test_parity_geometry as TG

pytestmark = pytest.mark.gpu


def _tune(pair):
    from paper_2510_21956_b200 import _abi
    t = _abi.Tuning()
    t.bwd_pair = pair
    _abi.lib().la_set_tuning(C.byref(t))


@pytest.fixture
def restore_tuning():
    yield
    from paper_2510_21956_b200 import _abi
    _abi.lib().la_set_tuning(None)


@pytest.mark.parametrize("G,N,groups", [(64, 2048, [0, 63]), (40, 4096, [5, 39]), (2, 1024, [1])])
def test_pair_backward_parity(cuda, restore_tuning, G, N, groups):
    t = TG.device_inputs(G, N, 128, seed=70 + G, cuda=cuda)
    _tune(-1)
    ref = [x.clone() for x in TG.device_step(*t)]
    _tune(1)
    res = TG.device_step(*t)
    TG.check_groups(f"pair_G{G}_N{N}", t, res, groups)
    for name, a, b in zip(("dq", "dk", "dv"), ref[2:], res[2:]):
        d = (a.float() - b.float()).abs().max().item()
        assert d <= 4e-3, (name, d)
    # the forward is shared: identical outputs
    assert (ref[0] == res[0]).all() and (ref[1] == res[1]).all()


def test_pair_backward_north_star_geometry(cuda, restore_tuning):
    t = TG.device_inputs(64, 65536, 128, seed=72, cuda=cuda)
    _tune(1)
    res = TG.device_step(*t)
    TG.check_groups("pair_G64_N65536", t, res, [0, 31, 63])


def test_pair_backward_is_deterministic(cuda, restore_tuning):
    t = TG.device_inputs(64, 4096, 128, seed=73, cuda=cuda)
    _tune(1)
    a = [x.clone() for x in TG.device_step(*t)]
    b = TG.device_step(*t)
    for x, y in zip(a[2:], b[2:]):
        assert (x == y).all()
