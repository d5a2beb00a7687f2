import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
L = _abi.lib()
dev = torch.device('cuda')
G, N, D = 64, int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 128
p = _abi.make_problem(G, N, D, "bf16")
q = torch.randn(G, N, D, device=dev); q = (q / q.norm(dim=-1, keepdim=True)).bfloat16()
k = q.clone(); v = (torch.rand(G, D, N, device=dev) * 2 - 1).bfloat16(); w = v.clone()
out = torch.empty(G, D, N, device=dev, dtype=torch.bfloat16); g = torch.empty(G, N, device=dev)
dq = torch.empty_like(q); dk = torch.empty_like(v); dv = torch.empty_like(v)
wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
for _ in range(2):
    L.la_forward(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), wsf.data_ptr(), wsf.numel(), None, None)
    L.la_backward(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), w.data_ptr(), 0, g.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), None, None)
torch.cuda.synchronize()
