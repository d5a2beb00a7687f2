"""North-star step with la_tuning.prefetch = PF (L2 prefetch distance of the sweeps' TMA rings)."""
import ctypes as C
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
t = TG.device_inputs(64, 65536, 128, seed=5, cuda=torch.device("cuda:0"))
for pf in [int(x) for x in sys.argv[1:]]:
    tu = _abi.Tuning()
    tu.prefetch = pf
    L.la_set_tuning(C.byref(tu))
    for _ in range(2):
        TG.device_step(*t)
    torch.cuda.synchronize()
    L.la_profile_enable(1)
    _abi.profile_read()
    for _ in range(5):
        TG.device_step(*t)
    torch.cuda.synchronize()
    per = {}
    for r in _abi.profile_read():
        per.setdefault(r["name"], []).append(r["ms"])
    L.la_profile_enable(0)
    print("pf", pf, {k: round(statistics.median(v), 4) for k, v in per.items()}, flush=True)
