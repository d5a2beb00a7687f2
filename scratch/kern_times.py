"""Per-kernel device times of one causal fwd+bwd (saved states) at G, N (median of 5)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
G, N = int(sys.argv[1]), int(sys.argv[2])
t = TG.device_inputs(G, N, 128, seed=5, cuda=torch.device("cuda:0"))
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
print(_abi.LIB_PATH[-18:], G, N, {k: round(statistics.median(v), 4) for k, v in per.items()},
      "sum", round(sum(statistics.median(v) for v in per.values()), 4))
