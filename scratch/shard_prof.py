"""One config-3 shard step (16 groups x 4096 rows) for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
from tests import test_parity_geometry as TG

t = TG.device_inputs(16, 4096, 128, seed=3, cuda=torch.device("cuda:0"))
for _ in range(4):
    TG.device_step(*t)
torch.cuda.synchronize()
