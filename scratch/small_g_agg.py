"""Config-3 shard (16 groups x 4096 rows): per-kernel times vs the aggregate unit split A."""
import ctypes as C
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
G, N = int(sys.argv[1]), int(sys.argv[2])
t = TG.device_inputs(G, N, 128, seed=3, cuda=torch.device("cuda:0"))
for A in [int(x) for x in sys.argv[3:]]:
    tu = _abi.Tuning()
    tu.agg_split = A
    L.la_set_tuning(C.byref(tu))
    for _ in range(3):
        TG.device_step(*t)
    torch.cuda.synchronize()
    L.la_profile_enable(1)
    _abi.profile_read()
    for _ in range(7):
        TG.device_step(*t)
    torch.cuda.synchronize()
    per = {}
    for r in _abi.profile_read():
        per.setdefault(r["name"], []).append(r["ms"])
    L.la_profile_enable(0)
    med = {k: round(statistics.median(v), 4) for k, v in per.items()}
    print("A", A, med, "sum", round(sum(med.values()), 4), flush=True)
