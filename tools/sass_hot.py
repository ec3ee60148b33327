"""Top SASS instructions by stall samples from `ncu --page source --csv --print-source sass`,
plus the instruction-count share per function-like region."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(lines[1:]))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
data = []
for idx, r in enumerate(rows[1:]):
    try:
        data.append((idx, r[1].strip(), int(r[si] or 0), int(r[ii] or 0)))
    except (ValueError, IndexError):
        pass
tot_s = sum(d[2] for d in data) or 1
tot_i = sum(d[3] for d in data) or 1
print(f"samples {tot_s}  warp-instructions {tot_i}")
for idx, src, s, i in sorted(data, key=lambda d: -d[2])[:n]:
    print(f"{idx:5d} {100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% ins  {src[:70]}")
