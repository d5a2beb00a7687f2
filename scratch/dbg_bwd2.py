import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from tests._util import fast_inputs, max_abs
from tests.test_parity_gpu import run_dev, oracle_all
from oracle import oracle as O
cuda = torch.device('cuda:0')
N = 64
q, k, v, w = fast_inputs(1, N, 128, seed=1)
res = run_dev(q, k, v, w, "bf16", cuda, impl="auto", impl_bwd="tcgen05")
qr, kr, vr = res["rounded"]; wr = res["w"]; g = res["g"]; o = res["out"]
what = wr / g[..., None]
s = (o * what).sum(-1)
T = np.tril(np.ones((N, N)))
dS = T * (what[0] @ vr[0].T - s[0][:, None])
term1 = dS @ kr[0]
print("term1 (dS K) ref", term1[:2, :4])
print("got", res["dq"][0, :2, :4])
print("err full", max_abs(res["dq"][0], term1))
S = kr[0].T @ vr[0]   # [m][j]
term2 = what[0] @ S.T
print("term1+term2 err", max_abs(res["dq"][0], term1 + term2), " term2 only err", max_abs(res["dq"][0], term2))
