"""fp32 fwd+bwd time: tensor-core (3xTF32) vs CUDA-core path, config 1 and larger shapes."""
import ctypes as C, sys, json
import torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi
L = _abi.lib()
dev = torch.device('cuda')
def run(G, N, D, impl, causal=True, iters=5, dt="f32"):
    p = _abi.make_problem(G, N, D, dt, 1.0, 1.0, causal, impl=impl)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    q = torch.randn(G, N, D, device=dev); q = (q / q.norm(dim=-1, keepdim=True)).to(tdt)
    k = q.roll(1, 1).contiguous(); v = (torch.rand(G, D, N, device=dev) * 2 - 1).to(tdt); w = (torch.rand(G, D, N, device=dev) * 2 - 1).to(tdt)
    out = torch.empty_like(v); g = torch.empty(G * N, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(v), torch.empty_like(v)
    wf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
    wb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), dtype=torch.uint8, device=dev)
    def step():
        assert L.la_forward(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), wf.data_ptr(), wf.numel(), None, None) == 0
        assert L.la_backward(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), w.data_ptr(), 0, g.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wb.data_ptr(), wb.numel(), None, None) == 0
    step(); torch.cuda.synchronize()
    L.la_profile_enable(1); _abi.profile_read()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(iters): step()
    t1.record(); torch.cuda.synchronize()
    prof = _abi.profile_read(); L.la_profile_enable(0)
    ks = {}
    for r in prof: ks[r["name"]] = ks.get(r["name"], 0) + r["ms"] / iters
    ms = t0.elapsed_time(t1) / iters
    byts = G * N * (12 * D * (4 if dt == "f32" else 2) + 8)  # fwd 4De+4 + bwd 8De+4
    print(json.dumps({"dt": dt, "G": G, "N": N, "D": D, "impl": impl, "causal": causal, "ms": round(ms, 4), "GB/s": round(byts / ms / 1e6, 1), "kernels": {a: round(b, 4) for a, b in ks.items()}}), flush=True)
import os
if os.environ.get("DT") == "bf16":
    for D in (32, 64, 128, 192, 256):
        run(64, 32768, D, "tcgen05", iters=3, dt="bf16")
    sys.exit(0)
for impl in ("tcgen05", "simt"):
    run(4, 2048, 64, impl)
    run(4, 2048, 64, impl, causal=False)
    run(16, 16384, 128, impl, iters=2)
run(64, 65536, 128, "tcgen05", iters=2)
run(64, 65536, 128, "tcgen05", causal=False, iters=2)
