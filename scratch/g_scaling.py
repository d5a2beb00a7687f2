"""bwd / fwd sweep time at G = 64 (128 CTAs) vs G = 74 (148 CTAs), P = 2: do the 20 idle
SMs add throughput, or is the sweep limited by shared HBM / L2 contention?"""
import os, sys
sys.path.insert(0, '.')
os.environ["LA_SEGMENTS"] = "2"
from paper_2510_21956_b200 import _abi, bench_csv as B
L = _abi.lib()
for H in (64, 74, 56):
    L.la_profile_enable(1); _abi.profile_read()
    B.run_sweep(1, H, (65536,), (128,), True, "bf16", repeats=5)
    per = {}
    for r in _abi.profile_read(): per.setdefault(r["name"], []).append(r["ms"])
    L.la_profile_enable(0)
    print(H, {k: round(sorted(v)[len(v) // 2], 4) for k, v in per.items()}, flush=True)
