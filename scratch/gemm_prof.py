import os, sys
sys.path.insert(0, '.')
from paper_2510_21956_b200 import bench_csv as B
D = int(os.environ.get("D", "256"))
B.run_sweep(2, 32, (32768,), (D,), False, "bf16", repeats=1)
