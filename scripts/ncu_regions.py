"""Aggregate an ncu SASS source page (csv) into source-line regions of one kernel.
usage: python scripts/ncu_regions.py <sass.csv> <cubin> <function-substring> <file> name:lo-hi ...
Lines of other files (inlined helpers) are attributed to the region of the call site when
nvdisasm reports it, else to 'other'."""
import csv, re, subprocess, sys
from collections import Counter

sass_csv, cubin, fsub, fname = sys.argv[1:5]
regions = []
for spec in sys.argv[5:]:
    n, r = spec.split(":")
    lo, hi = r.split("-")
    regions.append((n, int(lo), int(hi)))
dis = subprocess.run(["nvdisasm", "-g", "-gi", "-c", cubin], capture_output=True, text=True).stdout
lines = {}
cur_fn, cur = None, None
for ln in dis.splitlines():
    m = re.match(r"^\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "(.*?)", line (\d+)(.*)', ln)
    if m:
        f, l, rest = m.group(1).rsplit("/", 1)[-1], int(m.group(2)), m.group(3)
        # inlined-at chain: take the innermost location in fname
        chain = [(f, l)] + [(a.rsplit("/", 1)[-1], int(b)) for a, b in re.findall(r'inlined at "(.*?)", line (\d+)', rest)]
        sel = [c for c in chain if c[0] == fname]
        cur = sel[0] if sel else chain[0]
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and fsub in cur_fn:
        lines[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
ie, samp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[0], 16), int(r[ie] or 0), int(r[samp] or 0)) for r in rows[2:] if len(r) >= len(h)]
base = min(a for a, _, _ in data)
ci, cs = Counter(), Counter()
for a, n, s in data:
    f, l = lines.get(a - base, ("?", -1))
    reg = "other"
    if f == fname:
        for nm, lo, hi in regions:
            if lo <= l <= hi:
                reg = nm
                break
    ci[reg] += n
    cs[reg] += s
ti, ts = sum(ci.values()), sum(cs.values())
print(f"total instructions {ti:.3e}  stall samples {ts}")
for r, n in sorted(ci.items(), key=lambda kv: -kv[1]):
    print(f"{r:>12s} {100*n/ti:6.2f}% inst  {100*cs[r]/ts:6.2f}% samples")
