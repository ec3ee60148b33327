"""DRAM traffic and key counters per kernel from an ncu --set full report.

usage: python tools/ncu_traffic.py report.ncu-rep [more.ncu-rep ...]
Prints one line per profiled launch and a JSON dict {kernel: mean bytes}.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           # atomics (north_star: atomic throughput per kernel); captured with
           # --metrics next to --set full (tools/profile_round.sh)
           "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
           "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
         "ns": 1, "us": 1e3, "ms": 1e6}

per = defaultdict(list)
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        k = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        rec = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    rec[m] = float(r[i].replace(",", "")) * UNITS.get(units[i], 1)
                except ValueError:
                    pass
        per[k].append(rec)
summary = {}
for k, recs in per.items():
    mean = {m: sum(r.get(m, 0) for r in recs) / len(recs) for m in METRICS}
    traffic = mean["dram__bytes_read.sum"] + mean["dram__bytes_write.sum"]
    dur = mean["gpu__time_duration.sum"]
    atom = mean["lts__t_sectors_op_atom.sum"] + mean["lts__t_sectors_op_red.sum"]
    summary[k] = {"launches": len(recs), "duration_ns": dur, "dram_bytes": traffic,
                  "dram_gbs": traffic / dur if dur else 0.0,
                  "l2_hit_pct": mean["lts__t_sector_hit_rate.pct"],
                  "warps_active_pct": mean["sm__warps_active.avg.pct_of_peak_sustained_active"],
                  "regs": mean["launch__registers_per_thread"],
                  "l2_atom_sectors": mean["lts__t_sectors_op_atom.sum"],
                  "l2_red_sectors": mean["lts__t_sectors_op_red.sum"],
                  "l2_atomic_sectors_per_us": atom / (dur / 1e3) if dur else 0.0,
                  "l2_atomic_unit_busy_pct": mean["lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed"],
                  "fp64_pipe_pct": mean["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]}
    print(f"{k:34s} n={len(recs)} {dur / 1e3:8.1f} us  dram {traffic / 1e6:8.2f} MB ({traffic / dur if dur else 0:6.0f} GB/s)"
          f"  L2 hit {mean['lts__t_sector_hit_rate.pct']:5.1f}%  warps {mean['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f}%"
          f"  regs {mean['launch__registers_per_thread']:.0f}  atom+red {atom / 1e3:7.1f}K sect"
          f"  atomic unit {mean['lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed']:4.1f}%"
          f"  fp64 {mean['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']:4.1f}%")
print(json.dumps(summary))
