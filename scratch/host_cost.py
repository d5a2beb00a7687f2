"""Host-side cost of the C-ABI calls (no sync inside): config 1 (f32) and the north star."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()
dev = torch.device("cuda:0")
for (G, N, D, dt) in ((4, 2048, 64, "f32"), (16, 4096, 128, "bf16"), (64, 65536, 128, "bf16")):
    t = TG.device_inputs(G, N, D, seed=5, cuda=dev)
    if dt == "f32":
        t = [x.float() for x in t]
    q, k, v, w = t
    p = _abi.make_problem(G, N, D, dt)
    out = torch.empty_like(v); g = torch.empty((G, N), device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(v), torch.empty_like(v)
    wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    sv = torch.empty(max(1, L.la_saved_state_bytes(C.byref(p))), device=dev, dtype=torch.uint8)
    s = torch.cuda.current_stream().cuda_stream
    def fwd():
        return L.la_forward_save(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(),
                                 g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(), wsf.numel(), s, None)
    def bwd():
        return L.la_backward_saved(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(),
                                   w.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(), dq.data_ptr(),
                                   dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), s, None)
    for _ in range(3):
        fwd(); bwd()
    torch.cuda.synchronize()
    hf = hb = 0.0
    R = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(R):
        a = time.perf_counter(); fwd(); b = time.perf_counter(); bwd(); c = time.perf_counter()
        hf += b - a; hb += c - b
    e1.record()
    torch.cuda.synchronize()
    print(G, N, D, dt, "host us/call fwd", round(hf / R * 1e6, 1), "bwd", round(hb / R * 1e6, 1),
          "device ms/step", round(e0.elapsed_time(e1) / R, 4), flush=True)
