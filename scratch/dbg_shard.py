import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import sharding as S
from tests._util import fast_inputs
cuda = torch.device("cuda")
G, N, D = 3, 1024, 128
q, k, v, w = fast_inputs(G, N, D, seed=11)
tb = lambda x: torch.as_tensor(x).to(torch.bfloat16).to(cuda)
qs, ks = tb(q), tb(k)
vs, ws_ = tb(v.transpose(0, 2, 1)), tb(w.transpose(0, 2, 1))
for rep in range(3):
    tc, si = S.CudaOps(G, N, D, "bf16", impl="auto"), S.CudaOps(G, N, D, "bf16", impl="simt")
    f_tc, f_si = tc.forward_shard_state(ks, vs), si.forward_shard_state(ks, vs)
    out, g = tc.forward_with_carry(qs, ks, vs, torch.zeros_like(f_tc), 0)
    b_tc, b_si = tc.backward_shard_state(qs, out, ws_, g), si.backward_shard_state(qs, out, ws_, g)
    torch.cuda.synchronize()
    SZ = f_tc.numel() // G
    for name, a_, b_ in (("fwd", f_tc, f_si), ("bwd", b_tc, b_si)):
        a_, b_ = a_.double().cpu().numpy().reshape(G, SZ), b_.double().cpu().numpy().reshape(G, SZ)
        d = np.abs(a_ - b_)
        i = np.unravel_index(np.argmax(d), d.shape)
        print(rep, name, d.max(), i, a_[i], b_[i], "X max", np.abs(b_[:, :D*D]).max(), "vA", d[:, D*D:D*D+D].max(), "vB", d[:, D*D+D:D*D+2*D].max(), "cnt", a_[:, D*D+2*D], b_[:, D*D+2*D])
