"""fwd / bwd ms vs segment count for the small per-GPU problems (config 3 shards)."""
import os, sys
sys.path.insert(0, '.')
from paper_2510_21956_b200 import bench_csv as B
for (b, h, N) in ((2, 8, 4096), (4, 8, 4096), (8, 16, 4096), (1, 16, 131072)):
    for P in (1, 2, 3, 4, 6, 9, 12):
        os.environ["LA_SEGMENTS"] = str(P)
        r = B.run_sweep(b, h, (N,), (128,), True, "bf16", repeats=7)
        print(b * h, N, P, [round(x.wall_time_s * 1e3, 4) for x in r], round(sum(x.wall_time_s for x in r) * 1e3, 4), flush=True)
