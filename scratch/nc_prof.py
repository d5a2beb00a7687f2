import ctypes as C, json, sys, torch
sys.path.insert(0, '.')
from paper_2510_21956_b200 import _abi, bench_csv as B
L = _abi.lib()
L.la_profile_enable(1); _abi.profile_read()
B.run_sweep(2, 32, (32768,), (128,), False, "bf16", repeats=3)
per = {}
for r in _abi.profile_read(): per.setdefault(r["name"], []).append(r["ms"])
print({k: (round(sum(v) / len(v), 4), len(v)) for k, v in per.items()})
