"""Aggregate an ncu SASS source page (csv) per CUDA source line using nvdisasm -g line info.
usage: python scripts/ncu_lines.py <sass.csv> <cubin> <function-substring> [top]"""
import csv, re, subprocess, sys
from collections import Counter

sass_csv, cubin, fsub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines = {}
cur_fn, cur_line = None, None
for ln in dis.splitlines():
    m = re.match(r"^\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "(.*?)", line (\d+)', ln)
    if m:
        cur_line = (m.group(1).rsplit("/", 1)[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and fsub in cur_fn:
        lines[int(m.group(1), 16)] = cur_line
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
ie, samp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[0], 16), int(r[ie] or 0), int(r[samp] or 0)) for r in rows[2:] if len(r) >= len(h)]
base = min(a for a, _, _ in data)
ci, cs = Counter(), Counter()
for a, n, s in data:
    l = lines.get(a - base, ("?", -1))
    ci[l] += n
    cs[l] += s
ti, ts = sum(ci.values()), sum(cs.values())
print(f"total instructions {ti:.3e}  stall samples {ts}")
for l, n in sorted(ci.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{l[0]:>18s}:{l[1]:<5d} {100*n/ti:6.2f}% inst  {100*cs[l]/ts:6.2f}% stall")
