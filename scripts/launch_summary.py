"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel.
usage: python scripts/launch_summary.py launches.csv "command" "scope" > summary.txt"""
import collections
import csv
import re
import sys

path, cmd, scope = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    name = re.sub(r"^(void )?cfb::<unnamed>::", "", name)
    name = re.sub(r"\(.*$", "", name)
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}.get(d["Metric Unit"], 1e-6)
    tot[name] += float(d["Metric Value"].replace(",", "")) * scale
    cnt[name] += 1
T = sum(tot.values())
print("# ncu launch list summary (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)")
print(f"# command: {cmd}")
print(f"# scope: {scope}")
print(f"# launches: {sum(cnt.values())}  total kernel time: {T:.1f} ms")
print("# ms  share  launches  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.3f} {100 * v / T:5.1f}% {cnt[k]:6d}  {k[:100]}")
