"""Per-role clock64 timeline of the backward sweep (traced build, LA_CUDA_LIB)."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
L = _abi.lib()
dev = torch.device('cuda')
import os
if os.environ.get("PF"):
    tu = _abi.Tuning(); tu.prefetch = int(os.environ["PF"]); L.la_set_tuning(C.byref(tu))
G, N, D = 64, 65536, 128
p = _abi.make_problem(G, N, D, "bf16")
q = torch.randn(G, N, D, device=dev); q = (q / q.norm(dim=-1, keepdim=True)).bfloat16()
k = q.clone(); v = (torch.rand(G, D, N, device=dev) * 2 - 1).bfloat16(); w = v.clone()
out = torch.empty(G, D, N, device=dev, dtype=torch.bfloat16); g = torch.empty(G, N, device=dev)
dq = torch.empty_like(q); dk = torch.empty_like(v); dv = torch.empty_like(v)
wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
sv = torch.empty(L.la_saved_state_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
L.la_forward_save(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(), wsf.numel(), None, None)
for _ in range(3):
    L.la_backward_saved(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), w.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), None, None)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (4 * 64 * 10))()
L.la_internal_trace_read_bwd(buf)
t = np.array(buf, dtype=np.int64).reshape(4, 64, 10)
c0 = 20
t0 = t[0, c0, 0]
names = {0: "MMA  0:top 1:after ps/sR/gkv_empty 3:after sS/gq_empty 2:after full/dpt_empty(n+1)",
         1: "WG-A 0:dv_out start(after gkv_full) 1:after er_half 2:after e1_half",
         2: "WG-B 0:dq_out start(after gq_full) 1:E_S after waits 2:E_S done",
         3: "WG-C 0:after gkv_empty wait 1:after e1 2:end"}
for r in range(4):
    print(names[r])
    for c in range(c0, c0 + 4):
        print("  ", c, (t[r, c, :4] - t0).tolist())
print("period MMA top", np.diff(t[0, 10:60, 0]).mean())
for r, ev in ((1, 0), (1, 1), (1, 2), (2, 0), (2, 1), (2, 2), (3, 0), (3, 1), (3, 2), (0, 1), (0, 3), (0, 2), (0, 4), (3, 3), (0, 5), (0, 6), (3, 4), (3, 5), (3, 6), (3, 7), (2, 4)):
    x = t[r, 10:60, ev] - t[0, 10:60, 0]
    print(f"role {r} ev {ev}: mean offset vs MMA top {x.mean():.0f}")
