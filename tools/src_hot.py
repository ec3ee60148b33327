"""Per-source-line stall samples from `ncu --page source --csv --print-source cuda,sass`.

usage: ncu -i rep --page source --csv --kernel-name regex:K --print-source cuda,sass > f.csv
       python tools/src_hot.py f.csv [n]
"""
import csv
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = "?"
rows = []
hdr = None
with open(path) as fh:
    for rec in csv.reader(fh):
        if not rec:
            continue
        if rec[0] == "File Path":
            cur_file = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or rec[0] == "" or rec[0] == "Function Name":
            continue
        try:
            samples = int(rec[4] or 0)
            inst = int(rec[7] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((cur_file, rec[0], rec[1].strip(), samples, inst))
tot = sum(r[3] for r in rows) or 1
print(f"total samples {tot}")
for f, line, src, s, i in sorted(rows, key=lambda r: -r[3])[:n]:
    print(f"{100 * s / tot:5.1f}%  {f}:{line:>4s}  inst={i:>10d}  {src[:90]}")
