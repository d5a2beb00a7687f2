"""Per-kernel times of the north-star step for la_tuning settings given as key=value,... args."""
import ctypes as C
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
t = TG.device_inputs(64, 65536, 128, seed=5, cuda=torch.device("cuda:0"))
for rep in range(2):
    for spec in sys.argv[1:]:
        tu = _abi.Tuning()
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            setattr(tu, k, int(v))
        L.la_set_tuning(C.byref(tu))
        for _ in range(2):
            TG.device_step(*t)
        torch.cuda.synchronize()
        L.la_profile_enable(1)
        _abi.profile_read()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(5):
            TG.device_step(*t)
        ev[1].record()
        torch.cuda.synchronize()
        per = {}
        for r in _abi.profile_read():
            per.setdefault(r["name"], []).append(r["ms"])
        L.la_profile_enable(0)
        print(spec or "default", "step", round(ev[0].elapsed_time(ev[1]) / 5, 4),
              {k: round(statistics.median(v), 4) for k, v in per.items()}, flush=True)
