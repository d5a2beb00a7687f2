"""Measured fwd / bwd ms against the segment count P (LA_SEGMENTS) for B=4 H=16 D=128
bf16 causal at several N: calibrates choose_segments' cost model."""
import json, os, sys
sys.path.insert(0, '.')
from paper_2510_21956_b200 import bench_csv as B
res = {}
for N in (4096, 8192, 16384, 32768, 65536):
    for P in (1, 2, 3, 4, 5, 6, 8, 9, 12, 16):
        if N // 128 < P:
            continue
        os.environ["LA_SEGMENTS"] = str(P)
        r = B.run_sweep(4, 16, (N,), (128,), True, "bf16", repeats=5)
        res[f"{N}/{P}"] = [round(x.wall_time_s * 1e3, 4) for x in r]
        print(N, P, res[f"{N}/{P}"], flush=True)
json.dump(res, open("gpurun_out/seg_sweep.json", "w"))
