"""Config 1 (causal fp32 B1 H4 N2048 D64): per-kernel device times and the step time."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
G, N, D = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4, 2048, 64)))
dev = torch.device("cuda:0")
t = [x.float() for x in TG.device_inputs(G, N, D, seed=5, cuda=dev)]
for _ in range(3):
    TG.device_step(*t, dtype="f32")
torch.cuda.synchronize()
L.la_profile_enable(1)
_abi.profile_read()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10):
    TG.device_step(*t, dtype="f32")
ev[1].record()
torch.cuda.synchronize()
per = {}
for r in _abi.profile_read():
    per.setdefault(r["name"], []).append(r["ms"])
L.la_profile_enable(0)
print(G, N, D, "step(with host sync + allocs)", round(ev[0].elapsed_time(ev[1]) / 10, 4),
      {k: (round(statistics.median(v), 4), len(v) // 10) for k, v in per.items()},
      "sum", round(sum(statistics.median(v) * (len(v) // 10) for v in per.values()), 4))
