"""One bf16 generic-path forward (agg + scan + sweep) for ncu: G=64 N=32768 D=64 causal."""
import ctypes as C, sys
import torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
L = _abi.lib()
dev = torch.device('cuda')
G, N, D = 64, 32768, int(sys.argv[1]) if len(sys.argv) > 1 else 64
p = _abi.make_problem(G, N, D, "bf16", 1.0, 1.0, True, impl="tcgen05")
q = torch.randn(G, N, D, device=dev); q = (q / q.norm(dim=-1, keepdim=True)).bfloat16()
k = q.roll(1, 1).contiguous(); v = (torch.rand(G, D, N, device=dev) * 2 - 1).bfloat16()
out = torch.empty_like(v); g = torch.empty(G * N, device=dev)
wf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
assert L.la_forward(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), wf.data_ptr(), wf.numel(), None, None) == 0
torch.cuda.synchronize()
