"""Per-kernel times of one config-3 shard (16 groups x 4096 rows) under several segment counts."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
G, N = int(sys.argv[1]) if len(sys.argv) > 1 else 16, int(sys.argv[2]) if len(sys.argv) > 2 else 4096
t = TG.device_inputs(G, N, 128, seed=3, cuda=torch.device("cuda:0"))
for P in (0, 4, 8, 16, 32):
    tu = _abi.Tuning()
    tu.segments = P
    L.la_set_tuning(C.byref(tu))
    for _ in range(3):
        TG.device_step(*t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        TG.device_step(*t)
    e1.record()
    torch.cuda.synchronize()
    L.la_profile_enable(1)
    _abi.profile_read()
    for _ in range(5):
        TG.device_step(*t)
    torch.cuda.synchronize()
    prof = _abi.profile_read()
    L.la_profile_enable(0)
    per = {}
    for r in prof:
        per.setdefault(r["name"], []).append(r["ms"])
    print(f"P={P}: step {e0.elapsed_time(e1) / 20:.4f} ms (incl. host sync in device_step)",
          {k: round(sum(v) / len(v), 4) for k, v in per.items()}, flush=True)
