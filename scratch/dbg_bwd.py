import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2510_21956_b200 as la
from oracle import oracle as O
from tests._util import fast_inputs, max_abs
from tests.test_parity_gpu import run_dev, oracle_all
cuda = torch.device('cuda:0')
for N in (64, 128):
    for (a, b) in ((1.0, 0.0), (0.0, 1.0), (1.0, 1.0)):
        q, k, v, w = fast_inputs(1, N, 128, seed=1)
        if a == 0.0:
            q = np.abs(q); k = np.abs(k)  # keep g away from 0
        res = run_dev(q, k, v, w, "bf16", cuda, impl="auto", impl_bwd="tcgen05", a=a, b=b)
        ref = oracle_all(res, True, a, b)
        errs = {key: max_abs(res[key], ref[key]) for key in ("out", "dq", "dk", "dv")}
        print(N, a, b, {k_: round(v_, 4) for k_, v_ in errs.items()})
        if N == 64 and a == 1.0 and b == 1.0:
            for key in ("dq", "dk", "dv"):
                d = np.abs(res[key] - ref[key])[0]
                rows = np.where(d.max(axis=1) > 0.02)[0]
                cols = np.where(d.max(axis=0) > 0.02)[0]
                print(key, 'bad rows', rows[:20], len(rows), 'bad cols', cols[:20], len(cols))
                print(' got', res[key][0, :3, :4]); print(' ref', ref[key][0, :3, :4])
