"""Per-CTA throughput of the aggregate and main kernels when the grid does not fill
the GPU (G groups x P=9 segments): does an aggregate CTA pull more than its 1/148
share of HBM when fewer CTAs compete? (decides whether overlapping them pays)"""
import ctypes as C, json, os, sys
os.environ.setdefault("LA_SEGMENTS", "9")
sys.path.insert(0, '.')
import torch
from paper_2510_21956_b200 import _abi
L = _abi.lib()
dev = torch.device('cuda')
N, D = 65536, 128
for G in (4, 8, 16, 32, 64):
    p = _abi.make_problem(G, N, D, "bf16")
    q = torch.randn(G, N, D, device=dev); q = (q / q.norm(dim=-1, keepdim=True)).bfloat16()
    k = q.clone(); v = (torch.rand(G, D, N, device=dev) * 2 - 1).bfloat16(); w = v.clone()
    out = torch.empty(G, D, N, device=dev, dtype=torch.bfloat16); g = torch.empty(G, N, device=dev)
    dq = torch.empty_like(q); dk = torch.empty_like(v); dv = torch.empty_like(v)
    wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    wsb = torch.empty(L.la_backward_workspace_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    sv = torch.empty(L.la_saved_state_bytes(C.byref(p)), device=dev, dtype=torch.uint8)
    def step():
        L.la_forward_save(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), g.data_ptr(), sv.data_ptr(), sv.numel(), wsf.data_ptr(), wsf.numel(), None, None)
        L.la_backward_saved(C.byref(p), q.data_ptr(), 1, k.data_ptr(), 1, v.data_ptr(), 0, out.data_ptr(), w.data_ptr(), 0, g.data_ptr(), sv.data_ptr(), sv.numel(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), wsb.data_ptr(), wsb.numel(), None, None)
    for _ in range(3): step()
    torch.cuda.synchronize()
    L.la_profile_enable(1); _abi.profile_read()
    for _ in range(5): step()
    torch.cuda.synchronize()
    L.la_profile_enable(0)
    per = {}
    for r in _abi.profile_read(): per.setdefault(r["name"], []).append(r["ms"])
    rows = G * N
    ctas = G * 9
    bytes_ = {"la_fwd_agg": rows * 512 * 8 / 9, "la_fwd_causal": rows * 1028, "la_bwd_agg": rows * 1032, "la_bwd_causal": rows * 1796}
    res = {}
    for n_, v_ in per.items():
        ms = sum(v_) / len(v_)
        nct = ctas * (8 / 9 if n_ == "la_fwd_agg" else 1)
        res[n_] = dict(ms=round(ms, 4), tbps=round(bytes_[n_] / ms / 1e9, 3), gbps_per_cta=round(bytes_[n_] / ms / 1e6 / min(nct, 148) / max(1, nct / 148), 1))
    print(G, json.dumps(res), flush=True)
    del q, k, v, w, out, g, dq, dk, dv, wsf, wsb, sv
    torch.cuda.empty_cache()
