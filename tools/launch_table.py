"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
per = defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        per[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]) / 1000.0)
total = sum(sum(v) for v in per.values())
print(f"{'kernel':44s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}")
for n, v in sorted(per.items(), key=lambda x: -sum(x[1])):
    print(f"{n[:44]:44s} {len(v):8d} {sum(v) / len(v):9.1f} {100 * sum(v) / total:5.1f}%")
print(f"total {total:.1f} us over {sum(len(v) for v in per.values())} launches")
