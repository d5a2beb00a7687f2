import sys
sys.path.insert(0, '.')
from paper_2510_21956_b200 import bench_csv as B
B.run_sweep(4, 16, (65535,), (128,), True, "bf16", repeats=1)
