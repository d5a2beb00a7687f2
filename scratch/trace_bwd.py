import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
L = _abi.lib()
dev = torch.device('cuda')
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
for _ in range(2):
    L.la_backward_saved(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), w.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), None, None)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (4 * 64 * 10))()
L.la_internal_trace_read_bwd(buf)
t = np.array(buf, dtype=np.int64).reshape(4, 64, 10)
t0 = t[0, 10, 0]
ent, pro, fin = t[0, 63, 8], t[0, 63, 9], t[0, 63, 7]
print("prologue", pro - ent, "first chunk", t[0, 0, 1] - pro, "total", fin - ent)
t = t - t0
t[t < -10**9] = -1
R = range(10, 14)
names = {0: "MMA : blk n start, dKdV issue(n), T1/dPt issue(n), dQ issue(n)",
         1: "WG-A: gkv_full(n) seen, E_R half done, E1 half done",
         2: "WG-B: gq_full(n) seen, E_S start, E_S done",
         3: "WG-C: E1 start(n), E1 done(n), du done(n)"}
cols = {0: 4, 1: 3, 2: 3, 3: 3}
for role in range(4):
    print(names[role])
    for c in R: print(c, t[role, c, :cols[role]].tolist())
d = np.diff(t[0, 1:64, 1])
print("period", d.mean(), "by 8:", [int(d[i:i+8].mean()) for i in range(0, 62, 8)])
