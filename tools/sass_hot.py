"""Top SASS instructions of an ncu source-page CSV (--page source --csv --print-source sass):
by warp-stall samples (with the dominant stall reasons) and by shared-memory bank conflicts.
Usage: python tools/sass_hot.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1] if rows[0][0] != "Address" else rows[0]
data = [r for r in rows if len(r) == len(h) and r[0] != "Address"]
col = {c: i for i, c in enumerate(h)}
iW = col["Warp Stall Sampling (All Samples)"]
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iW] or 0) for r in data)
print(f"total samples {tot:.0f}")
for k, r in sorted(enumerate(data), key=lambda x: -float(x[1][iW] or 0))[:n]:
    w = float(r[iW] or 0)
    st = sorted(((float(r[col[c]] or 0), c[6:]) for c in stalls), reverse=True)[:3]
    print(f"{k:5d} {w / tot * 100:5.2f}% {r[col['Source']][:70]:70s} " + " ".join(f"{c}={v / max(w, 1) * 100:.0f}%" for v, c in st))
print("--- shared conflicts (excess wavefronts)")
iC = col.get("L1 Wavefronts Shared Excessive")
if iC is not None:
    for k, r in sorted(enumerate(data), key=lambda x: -float(x[1][iC] or 0))[:15]:
        print(f"{k:5d} excess={r[iC]:>10} total={r[col['L1 Wavefronts Shared']]:>10} {r[col['Source']][:80]}")
