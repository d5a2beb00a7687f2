"""fp32 tensor-core path debug: per-case relative errors vs the f64 oracle."""
import sys
import numpy as np
sys.path.insert(0, '.')
from tests._util import fast_inputs, rel_err
from tests.test_parity_gpu import oracle_all, run_dev
import torch
cuda = torch.device('cuda')
for (G, N, D, causal) in [(1, 64, 128, True), (1, 64, 64, True), (1, 128, 128, True), (1, 64, 128, False), (1, 128, 128, False), (4, 2048, 64, True)]:
    q, k, v, w = fast_inputs(G, N, D, seed=1)
    res = run_dev(q, k, v, w, "f32", cuda, causal=causal, impl="tcgen05")
    ref = oracle_all(res, causal)
    errs = {kk: rel_err(res[kk], ref[kk]) for kk in ("out", "g", "dq", "dk", "dv")}
    print(G, N, D, causal, {kk: f"{e:.2e}" for kk, e in errs.items()})
    if errs["out"] > 1e-5:
        d = np.abs(res["out"] - ref["out"])[0]
        print("  out err by row (first 8 rows max):", d.max(1)[:8], " by feature (first 8):", d.max(0)[:8])
        print("  worst row/feature", np.unravel_index(np.argmax(d), d.shape), "dev", res["out"][0].flat[np.argmax(d)], "ref", ref["out"][0].flat[np.argmax(d)])
