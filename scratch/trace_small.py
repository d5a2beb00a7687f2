"""Prologue / loop / tail split of the backward sweep at small G (traced side library)."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG
L = _abi.lib()
G, N = int(sys.argv[1]), int(sys.argv[2])
t = TG.device_inputs(G, N, 128, seed=5, cuda=torch.device("cuda:0"))
for _ in range(3):
    TG.device_step(*t)
buf = (C.c_ulonglong * (4 * 64 * 10))()
L.la_internal_trace_read_bwd(buf)
x = np.array(buf, dtype=np.int64).reshape(4, 64, 10)
t0 = x[0, 63, 8]
print("start->carries loaded", x[0, 63, 9] - t0, "start->end", x[0, 63, 7] - t0)
for n in range(0, 9):
    print(n, "MMA top", x[0, n, 0] - t0, "stage landed", x[2, n, 4] - t0, "dKdV issue", x[0, n, 1] - t0)
