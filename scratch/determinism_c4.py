"""Run-to-run determinism of one fwd+bwd at the config-4 geometry (non-causal G=64 N=32768)
for the library in LA_CUDA_LIB: R repeats on the same inputs, outputs compared bitwise
against the first; for a mismatch print which tensor, how many elements, which groups/rows."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

cuda = torch.device("cuda:0")
D = int(sys.argv[1]) if len(sys.argv) > 1 else 64
R = int(sys.argv[2]) if len(sys.argv) > 2 else 20
causal = len(sys.argv) > 3 and sys.argv[3] == "causal"
fwd_only = len(sys.argv) > 3 and sys.argv[3] == "fwd"
G, N = (64, 32768) if not causal else (64, 65536)
t = TG.device_inputs(G, N, D, seed=3, cuda=cuda)
def step():
    if not fwd_only:
        return TG.device_step(*t, causal=causal)
    import ctypes as C
    from paper_2510_21956_b200.api import _raise
    L = _abi.lib()
    q, k, v, w = t
    p = _abi.make_problem(G, N, D, "bf16", 1.0, 1.0, False)
    out = torch.empty_like(v)
    g = torch.empty((G, N), device=cuda, dtype=torch.float32)
    wsf = torch.empty(L.la_forward_workspace_bytes(C.byref(p)), device=cuda, dtype=torch.uint8)
    err = _abi.ErrorInfo()
    _raise(L.la_forward(C.byref(p), q.data_ptr(), TG.SM, k.data_ptr(), TG.SM, v.data_ptr(), TG.FM, out.data_ptr(),
                        g.data_ptr(), wsf.data_ptr(), wsf.numel(), torch.cuda.current_stream().cuda_stream,
                        C.byref(err)), err)
    torch.cuda.synchronize()
    return out, g


ref = [x.clone() for x in step()]
names = ["out", "g", "dq", "dk", "dv"]
bad = 0
for it in range(R):
    res = step()
    for nm, a, b in zip(names, ref, res):
        ne = (a.view(torch.uint8) != b.view(torch.uint8)) if a.dtype != torch.float32 else (a != b)
        if ne.any():
            bad += 1
            idx = ne.nonzero()
            grps = sorted(set(idx[:, 0].tolist()))[:10]
            d = (a.float() - b.float()).abs().max().item()
            print(f"iter {it} {nm}: {int(ne.sum())} elements differ, groups {grps}, first {idx[0].tolist()}, max diff {d:.3e}", flush=True)
print(f"D={D} causal={causal} fwd_only={fwd_only} repeats={R} mismatching tensors: {bad}", flush=True)
