"""Where do the pair backward's dq values differ from the single-CTA sweep? (race hunting)"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()


def tune(pair):
    t = _abi.Tuning()
    t.bwd_pair = pair
    L.la_set_tuning(C.byref(t))


G, N = int(sys.argv[1]), int(sys.argv[2])
t = TG.device_inputs(G, N, 128, seed=7, cuda=torch.device("cuda:0"))
tune(-1)
ref = TG.device_step(*t)[2].float()
tune(1)
for rep in range(4):
    dq = TG.device_step(*t)[2].float()
    d = (dq - ref).abs()
    bad = (d > 1e-2).nonzero()
    print(f"rep {rep}: max {d.max().item():.3e}, bad elements {bad.shape[0]}", flush=True)
    if bad.shape[0]:
        rows = bad[:, 1]
        grp = bad[:, 0]
        print("   groups", torch.unique(grp).tolist()[:20], " rows", torch.unique(rows).tolist()[:40],
              " chunks(64)", torch.unique(rows // 64).tolist()[:20], " cols", torch.unique(bad[:, 2]).tolist()[:16])
