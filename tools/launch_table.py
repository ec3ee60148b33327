"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel.

Kernels of fa_set_mesh (per mesh, not per frame: index check, Morton order,
renumbering, cluster data) and torch's own are listed apart from the frame's."""
import csv
import sys
from collections import defaultdict

PER_MESH = ("k_ms_", "k_rs_", "k_mesh_", "k_cluster_build", "k_first_use", "k_permute_pos", "k_fill")

path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
per = defaultdict(list)
for r in rows:
    if r["Metric Name"] == "gpu__time_duration.sum":
        per[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]) / 1000.0)


def group(name):
    n = name.replace("void ", "")
    if n.startswith(PER_MESH):
        return "per mesh (fa_set_mesh)"
    if not n.startswith("k_"):
        return "other (torch)"
    return "per frame"


for g in ("per frame", "per mesh (fa_set_mesh)", "other (torch)"):
    items = {n: v for n, v in per.items() if group(n) == g}
    if not items:
        continue
    total = sum(sum(v) for v in items.values())
    print(f"== {g}")
    print(f"{'kernel':44s} {'launches':>8s} {'mean_us':>9s} {'share':>6s}")
    for n, v in sorted(items.items(), key=lambda x: -sum(x[1])):
        print(f"{n[:44]:44s} {len(v):8d} {sum(v) / len(v):9.1f} {100 * sum(v) / total:5.1f}%")
    print(f"total {total:.1f} us over {sum(len(v) for v in items.values())} launches\n")
