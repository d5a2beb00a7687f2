"""la_host_step time at the north star for la_tuning.host_blocks values given as args."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi

L = _abi.lib()
G, N, D = 64, 65536, 128
p = _abi.make_problem(G, N, D, "bf16")
pin = dict(dtype=torch.bfloat16, pin_memory=True)
hq, hk = torch.empty((G, N, D), **pin), torch.empty((G, N, D), **pin)
hv, hw = torch.empty((G, D, N), **pin), torch.empty((G, D, N), **pin)
for x in (hq, hk, hv, hw):
    x.uniform_(-1, 1)
hq /= hq.float().norm(dim=-1, keepdim=True).bfloat16()
hk /= hk.float().norm(dim=-1, keepdim=True).bfloat16()
hout, hdq, hdk, hdv = (torch.empty(x.shape, **pin) for x in (hv, hq, hv, hv))
hg = torch.empty((G, N), dtype=torch.float32, pin_memory=True)
err = _abi.ErrorInfo()
for rep in range(2):
    for hb in [int(x) for x in sys.argv[1:]]:
        tu = _abi.Tuning(); tu.host_blocks = hb; L.la_set_tuning(C.byref(tu))
        def step():
            st = L.la_host_step(C.byref(p), hq.data_ptr(), 1, hk.data_ptr(), 1, hv.data_ptr(), 0, hw.data_ptr(), 0,
                                hout.data_ptr(), hg.data_ptr(), hdq.data_ptr(), hdk.data_ptr(), hdv.data_ptr(),
                                C.byref(err))
            assert st == 0, err.message
        step()
        t0 = time.perf_counter()
        for _ in range(3):
            step()
        print("host_blocks", hb, round((time.perf_counter() - t0) / 3 * 1e3, 2), "ms", flush=True)
