import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
L = _abi.lib()
dev = torch.device('cuda')
G, N, D = 64, 65536, 128
p = _abi.make_problem(G, N, D, "bf16")
q = torch.randn(G, N, D, device=dev).bfloat16(); q /= q.float().norm(dim=-1, keepdim=True).bfloat16()
k = q.clone(); v = torch.rand(G, D, N, device=dev).bfloat16()
out = torch.empty(G, D, N, device=dev, dtype=torch.bfloat16); g = torch.empty(G, N, device=dev)
ws = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
for _ in range(3):
    L.la_forward(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), ws.data_ptr(), ws.numel(), None, None)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (4 * 64 * 8))()
L.la_internal_trace_read(buf)
t = np.array(buf, dtype=np.int64).reshape(4, 64, 8)
t0 = t[0, 10, 0]
t = t - t0
t[t < -10**9] = -1
R = range(8, 14)
print("MMA  : start, sb_ready, p_ready, ot_empty(M2 issue), T1(c+1) issued")
for c in R: print(c, t[0, c, [0, 1, 4, 5, 2]].tolist())
print("WG-S : E2start, sb_ready arrive, st_full(c)")
for c in R: print(c, t[1, c, :3].tolist())
print("WG-A : t1_full, T1 loaded, g/a2b, o_full(c-2), p_ready")
for c in R: print(c, t[1, c, [3, 7, 4, 5, 6]].tolist())
print("WG-B : start, o_full, a2b, ot_empty, store")
for c in R: print(c, t[2, c, :5].tolist())
print("PROD : start, empty")
for c in R: print(c, t[3, c, :2].tolist())
print("period", np.diff(t[0, 5:60, 0]).mean())
