"""One north-star fwd+bwd with the pair backward (for ncu captures)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
t = _abi.Tuning()
t.bwd_pair = int(sys.argv[1]) if len(sys.argv) > 1 else 1
L.la_set_tuning(C.byref(t))
G = int(sys.argv[2]) if len(sys.argv) > 2 else 64
x = TG.device_inputs(G, 65536, 128, seed=7, cuda=torch.device("cuda:0"))
for _ in range(3):
    TG.device_step(*x)
torch.cuda.synchronize()
