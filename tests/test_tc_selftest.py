"""Hardware self-test of the tcgen05 building blocks (tests/csrc/tc_selftest.cu):
UMMA descriptors in K-major / MN-major SW128, A operand from TMEM, TMEM ld/st and
TMA 3D loads, each checked against a float64 matmul."""
import ctypes as C
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "csrc", "libtc_selftest.so")

pytestmark = pytest.mark.gpu

MODES = {0: "A K-major smem, B K-major smem", 1: "A MN-major smem", 2: "B MN-major smem",
         3: "A from TMEM", 4: "TMA 3D loads (SW128)", 5: "M=64 into upper lane half",
         6: "M=64 A MN-major negated"}


@pytest.mark.parametrize("mode", sorted(MODES))
def test_umma_building_block(cuda, mode):
    import torch
    lib = C.CDLL(LIB)
    g = torch.Generator().manual_seed(mode)
    A = (torch.rand(128, 128, generator=g) * 2 - 1).to(torch.bfloat16)
    B = (torch.rand(128, 128, generator=g) * 2 - 1).to(torch.bfloat16)
    dA, dB = A.to(cuda), B.to(cuda)
    D = torch.zeros(128, 128, dtype=torch.float32, device=cuda)
    rc = lib.tc_selftest(C.c_void_p(dA.data_ptr()), C.c_void_p(dB.data_ptr()), C.c_void_p(D.data_ptr()),
                         C.c_int(mode))
    assert rc == 0, f"CUDA error {rc}"
    ref = A.double().numpy() @ B.double().numpy().T
    got = D.cpu().double().numpy()
    if mode >= 5:
        ref = ref[:64, :64] * (-1.0 if mode == 6 else 1.0)
        got = got[:64, :64]
    err = np.abs(got - ref).max()
    assert err < 1e-3, (MODES[mode], err)
