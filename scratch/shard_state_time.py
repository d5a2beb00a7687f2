import sys, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import sharding as S
G, N, D = 16, 131072, 128
dev = torch.device("cuda")
q = torch.randn(G, N, D, device=dev); q = (q / q.norm(dim=-1, keepdim=True)).bfloat16()
k = q.clone(); v = (torch.rand(G, D, N, device=dev) * 2 - 1).bfloat16(); w = v.clone()
for impl in ("auto", "simt"):
    ops = S.CudaOps(G, N, D, "bf16", impl=impl)
    st = ops.forward_shard_state(k, v)
    out, g = ops.forward_with_carry(q, k, v, torch.zeros_like(st), 0)
    for name, fn in (("fwd_state", lambda: ops.forward_shard_state(k, v)), ("bwd_state", lambda: ops.backward_shard_state(q, out, w, g))):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        print(impl, name, round(a.elapsed_time(b), 3), "ms", flush=True)
