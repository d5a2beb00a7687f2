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
t0 = t[3, 0, 0]
names = {0: "MMA: start,sb_ready,full(c+1),t1_empty,p_ready,ot_empty", 1: "WGA: E2start,st_full,sbready,t1_full,a2b/empty,o_full(c-1),p_ready",
         2: "WGB: start,o_full,a2b,ot_empty,store_issued,store_read", 3: "PROD: start,empty"}
for role in range(4):
    print(names[role])
    for c in range(10, 16):
        print(c, (t[role, c] - t0).tolist())
print("per-chunk period (MMA start):", np.diff(t[0, 5:60, 0]).mean())
print("WGA fine: t1_full, after T1 loads, after dot+g, after named_bar, after z(empty)")
for c in range(10, 16): print(c, (t[1, c, [3, 7]] - t0).tolist(), (t[2, c, [6, 7]] - t0).tolist(), (t[1, c, 4] - t0))
