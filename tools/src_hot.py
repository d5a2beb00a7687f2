"""Top CUDA source lines by warp-stall samples from an ncu source CSV exported with
--page source --csv --print-source cuda,sass. Usage: python tools/src_hot.py file.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out, fname, hdr = [], "?", None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {c: i for i, c in enumerate(r)}
        continue
    if hdr is None or len(r) < 5 or r[2] != "-":
        continue
    w = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    if w <= 0:
        continue
    stalls = sorted(((float(r[i] or 0), c[6:]) for c, i in hdr.items()
                     if c.startswith("stall_") and "Not Issued" not in c), reverse=True)[:3]
    out.append((w, fname, r[0], r[1].strip(), stalls))
tot = sum(o[0] for o in out)
for w, f, ln, src, st in sorted(out, reverse=True)[:n]:
    print(f"{w / tot * 100:5.1f}% {f}:{ln:5s} {src[:75]:75s} " + " ".join(f"{c}={v / w * 100:.0f}%" for v, c in st))
