"""Pipeline trace of the pair backward (scratch/libla_trace.so, built by scratch/build_trace.sh):
per role and chunk, cycles spent waiting vs working (clock64, per CTA)."""
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
G = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x = TG.device_inputs(G, 65536, 128, seed=7, cuda=torch.device("cuda:0"))
for _ in range(2):
    TG.device_step(*x)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (2 * 5 * 64 * 4))()
L.la_internal_trace_read_pair(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(2, 5, 64, 4).astype(np.int64)
names = {0: ["MMA", "WG-A e1/dv", "WG-B er/dk", "WG-C dc/e1/du", "ring"],
         1: ["MMA", "WG-A E0", "WG-B E_S", "WG-C e1/zs/dq", "producer"]}
for rank in (0, 1):
    base = a[rank][a[rank] > 0].min()
    print(f"== rank {rank} ({'KV' if rank == 0 else 'Q'}) chunk period (cycles):",
          np.diff(a[rank, 0, :, 1]).mean() if rank == 0 else np.diff(a[rank, 0, :, 1]).mean())
    for role in range(5):
        ev = a[rank, role]
        if not ev.any():
            continue
        rel = ev - base
        d = np.diff(ev, axis=1)
        print(f"  {names[rank][role]:16s} ev-deltas mean {d[4:60].mean(0).round(0)}  period {np.diff(ev[:, 0])[4:60].mean():.0f}  (E0 sub: loop-end - ev2 of E0)" if False else f"  {names[rank][role]:16s} ev-deltas mean {d[4:60].mean(0).round(0)}  period {np.diff(ev[:, 0])[4:60].mean():.0f}")
        for n in (10, 11):
            print(f"     chunk {n}: {rel[n].tolist()}")
e0 = a[1, 1]
sub = a[1, 4]
print("E0 split (cycles): kvfree->loop end", (sub[4:60, 2] - e0[4:60, 2]).mean(), " loop end->s stored", (sub[4:60, 3] - sub[4:60, 2]).mean(),
      " s stored->pushed", (e0[4:60, 3] - sub[4:60, 3]).mean())
