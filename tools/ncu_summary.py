"""Per-kernel summary of an ncu --set full report: time, dram, L2 hit,
occupancy, IPC-ish counters and the top stall reasons.

usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]
"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
# ncu's second row holds each column's unit (byte / Kbyte / Mbyte, nsecond /
# usecond ...): values are scaled to bytes and microseconds here
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
         "ns": 1e-3, "us": 1, "ms": 1e3}


def get(row, key):
    i = col.get(key)
    if i is None:
        return None
    try:
        return float(row[i].replace(",", "")) * SCALE.get(units[i], 1)
    except ValueError:
        return None


for row in rows[2:]:
    name = row[col["Kernel Name"]].split("(")[0]
    if pat and not pat.search(name):
        continue
    t = get(row, "gpu__time_duration.sum")
    dram = (get(row, "dram__bytes_read.sum") or 0) + (get(row, "dram__bytes_write.sum") or 0)
    stalls = {}
    for h, i in col.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(row[i])
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1
    top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:4])
    print(f"{name:28s} {t:8.1f} us  dram {dram / 1e6:7.2f} MB  L2hit {get(row, 'lts__t_sector_hit_rate.pct') or 0:5.1f}%"
          f"  warps {get(row, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0:5.1f}%"
          f"  regs {get(row, 'launch__registers_per_thread') or 0:3.0f}"
          f"  inst {(get(row, 'smsp__inst_executed.sum') or 0) / 1e6:6.2f}M"
          f"  thr/inst {get(row, 'smsp__thread_inst_executed_per_inst_executed.ratio') or 0:5.1f}"
          f"  fp64 {get(row, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active') or 0:4.1f}%")
    print(f"{'':28s} stalls: {top}")
