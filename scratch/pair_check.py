"""Pair backward (la_bwd_pair.cu) against the single-CTA sweep: same inputs, outputs compared,
both timed (CUDA events), then sampled groups against the f64 chunked oracle."""
import ctypes as C
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_21956_b200 import _abi
from tests import test_parity_geometry as TG

L = _abi.lib()


def tune(pair):
    t = _abi.Tuning()
    t.bwd_pair = pair
    L.la_set_tuning(C.byref(t))


def run(G, N, groups, reps=5):
    cuda = torch.device("cuda:0")
    t = TG.device_inputs(G, N, 128, seed=7, cuda=cuda)
    res = {}
    for pair in (-1, 1):
        tune(pair)
        r = TG.device_step(*t)
        res[pair] = [x.clone() for x in r]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.la_profile_enable(1)
        _abi.profile_read()
        for _ in range(reps):
            TG.device_step(*t)
        torch.cuda.synchronize()
        prof = _abi.profile_read()
        L.la_profile_enable(0)
        per = {}
        for rr in prof:
            per.setdefault(rr["name"], []).append(rr["ms"])
        print(f"G={G} N={N} pair={pair}:", {k: round(sum(v) / len(v), 4) for k, v in per.items()}, flush=True)
    for i, name in enumerate(["out", "g", "dq", "dk", "dv"]):
        a, b = res[-1][i].float(), res[1][i].float()
        d = (a - b).abs().max().item()
        print(f"  {name}: max|old-pair| = {d:.3e}  max|old| = {a.abs().max().item():.3e}", flush=True)
    tune(1)
    w = TG.check_groups(f"pair_G{G}_N{N}", t, res[1], groups)
    print("  vs f64 oracle (pair):", {k: f"{v:.2e}" for k, v in w.items()}, flush=True)


if __name__ == "__main__":
    for G, N, groups in [(64, 2048, [0, 63]), (40, 4096, [5]), (64, 65536, [0, 37])]:
        run(G, N, groups)
