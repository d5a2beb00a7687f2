"""Hash of one causal fwd+bwd's outputs (saved and recomputed prefixes) at a few G, N for the
library in LA_CUDA_LIB: two libraries that must agree bitwise print the same lines."""
import hashlib
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

cuda = torch.device("cuda:0")
for G, N in ((64, 65536), (16, 4096), (3, 8192), (2, 1024)):
    t = TG.device_inputs(G, N, 128, seed=7, cuda=cuda)
    for saved in (True, False):
        outs = TG.device_step(*t, saved=saved)
        h = hashlib.sha1()
        for x in outs[2:]:
            h.update(x.contiguous().view(torch.uint8).cpu().numpy().tobytes())
        print(G, N, saved, h.hexdigest()[:16], flush=True)
    del t
