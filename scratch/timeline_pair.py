"""Cross-CTA timeline (globaltimer ns) of the pair backward for a few chunks of cluster 0."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
_abi.LIB_PATH = "scratch/libla_trace.so"
from tests import test_parity_geometry as TG

L = _abi.lib()
t = _abi.Tuning()
t.bwd_pair = 1
L.la_set_tuning(C.byref(t))
x = TG.device_inputs(64, 65536, 128, seed=7, cuda=torch.device("cuda:0"))
for _ in range(2):
    TG.device_step(*x)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (2 * 5 * 64 * 4))()
L.la_internal_trace_read_pair(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 5, 64, 4).astype(np.int64)
names = {(0, 0): ["KV-MMA wait sR/R+=", "KV-MMA dKdV issue", "KV-MMA td wait", "KV-MMA td issue"],
         (0, 1): ["KV-A e1 start", "KV-A e1 go", "KV-A dv go", "KV-A dv done"],
         (0, 2): ["KV-B er start", "KV-B er go", "KV-B er done", "KV-B dk done"],
         (0, 3): ["KV-C start", "KV-C wfull", "KV-C e1 done", "KV-C du done"],
         (0, 4): ["KV-3 acked", "KV-3 wempty", "-", "-"],
         (1, 0): ["Q-MMA wait sS", "Q-MMA dQ issue", "Q-MMA s/dpt next", "Q-MMA dpt issue"],
         (1, 1): ["Q-E0 start", "Q-E0 full", "Q-E0 kvfree", "Q-E0 pushed"],
         (1, 2): ["Q-ES start", "Q-ES s_full", "Q-ES dq_full", "Q-ES done"],
         (1, 3): ["-", "Q-C zs start", "Q-C zs done", "Q-C dq done"],
         (1, 4): ["Q-prod wait", "Q-prod go", "E0 loop end", "E0 s stored"]}
base = a[:, :, 20, :][a[:, :, 20, :] > 1e12].min()
ev = []
for (rank, role), nm in names.items():
    for n in (20, 21, 22):
        for e in range(4):
            v = a[rank, role, n, e]
            if v > 1e12 and nm[e] != "-":
                ev.append((v - base, n, nm[e]))
for v, n, nm in sorted(ev):
    print(f"{v:8d} ns  chunk {256 + n}  {nm}")
