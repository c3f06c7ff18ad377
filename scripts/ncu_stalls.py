"""Per-SASS-instruction stall breakdown from an ncu source page csv (--print-source sass).
usage: python scripts/ncu_stalls.py <sass.csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ix = {c: h.index(c) for c in cols}
ie = h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    st = {c: int(r[ix[c]] or 0) for c in cols}
    data.append((sum(st.values()), r[0], r[1], int(r[ie] or 0), st))
tot = sum(d[0] for d in data)
print(f"total samples {tot}")
for s, a, src, n, st in sorted(data, key=lambda d: -d[0])[:top]:
    parts = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    ps = " ".join(f"{k[6:]}={100 * v / max(s, 1):.0f}%" for k, v in parts if v)
    print(f"{100 * s / tot:5.2f}% {a[-5:]} {n:11d} {src[:52]:52s} {ps}")
