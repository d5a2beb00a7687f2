"""Per-region stall breakdown of an ncu SASS source CSV, regions delimited by clock64 reads."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = [r for r in rows[2:] if len(r) == len(h)]
iS = h.index('Source'); iW = h.index('Warp Stall Sampling (All Samples)'); iE = h.index('Instructions Executed')
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot = sum(float(r[iW] or 0) for r in data)
cuts = [0] + [k for k, r in enumerate(data) if 'SR_CLOCKLO' in r[iS]] + [len(data)]
for a, b in zip(cuts, cuts[1:]):
    seg = data[a:b]
    w = sum(float(r[iW] or 0) for r in seg)
    if w < tot * 0.01: continue
    st = {c: sum(float(r[h.index(c)] or 0) for r in seg) for c in cols}
    top = sorted(st.items(), key=lambda x: -x[1])[:4]
    ex = max(int(r[iE] or 0) for r in seg)
    print(f"[{a:5d},{b:5d}) {w/tot*100:5.1f}% maxexec={ex:8d} " + " ".join(f"{c[6:]}={v/w*100:.0f}%" for c, v in top))
print("cut labels (role, ev) from the trace STG offsets:")
import re
for k, r in enumerate(data):
    if 'SR_CLOCKLO' in r[iS]:
        lab = '?'
        for j in range(k + 1, min(k + 12, len(data))):
            m = re.search(r'STG\.E\.64 .*\+(0x[0-9a-f]+)\]', data[j][iS])
            if m:
                off = int(m.group(1), 16); lab = f"role{off // 5120} ev{(off % 5120) // 8}"; break
        print(k, lab)
