import sys
sys.path.insert(0, '.')
from paper_2510_21956_b200 import bench_csv as B
for N in (65536, 65535, 65472):
    r = B.run_sweep(4, 16, (N,), (128,), True, "bf16", repeats=3)
    print(N, [round(x.wall_time_s * 1e3, 3) for x in r], flush=True)
