"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel family.
usage: python scripts/launch_shares.py launches.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
kn, val = h.index("Kernel Name"), h.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    name = r[kn]
    m = re.search(r"(k_\w+)", name)
    if m:
        key = m.group(1)
        if key == "k_raster":
            key += "<render>" if "(bool)1" in name.split(",")[0] else "<score>"
    elif "cub" in name or "DeviceRadix" in name or "DeviceScan" in name:
        key = "cub " + re.sub(r".*?(Device\w+?Kernel|\w+Kernel).*", r"\1", name)[:40]
    else:
        key = name[:50]
    tot[key] += float(r[val].replace(",", "")) / 1e6
    cnt[key] += 1
T = sum(tot.values())
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / T:.1f}% |")
