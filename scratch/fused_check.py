"""One fused-schedule backward (la_tuning.bwd_fused = 1) at G, N; prints the time."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG
G, N = int(sys.argv[1]), int(sys.argv[2])
t = TG.device_inputs(G, N, 128, seed=5, cuda=torch.device("cuda:0"))
TG.device_step(*t); torch.cuda.synchronize()
_abi.set_tuning(bwd_fused=1)
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    t0 = time.time(); TG.device_step(*t); torch.cuda.synchronize()
    print("fused ok", i, G, N, round(time.time() - t0, 4), flush=True)
