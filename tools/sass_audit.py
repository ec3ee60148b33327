"""SASS audit of the product library: per-kernel opcode counts for the
instructions DESIGN.md's claims rest on, plus short excerpts.

  python tools/sass_audit.py [lib.so] > profiles/r2_sass_audit.txt

Counted (static instructions in each kernel's SASS):
  REDG.E.MIN.64   fire-and-forget 64-bit min reductions (depth keys / winners)
  ATOMG / REDG    other global atomics / reductions
  UBLKCP          cp.async.bulk (TMA engine) copies, SYNCS.* their mbarrier ops
  LDGSTS          cp.async (Ampere-style) global->shared copies
  DFMA/DADD/DMUL  FP64 arithmetic (DFMA: the OpenBLAS FMA chains, and inside the
                  correctly rounded division / square-root sequences)
  MUFU.RCP64H     FP64 reciprocal seeds (span reciprocals, division fast paths)
  BAR / WARPSYNC  block barriers
  ACQBULK / griddepcontrol: programmatic dependent launch (PDL) wait
"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2502_17712_b200/libfastatlas.so"
KEYS = ["REDG.E.MIN.64", "REDG", "ATOMG", "ATOMS", "UBLKCP", "SYNCS", "LDGSTS", "DFMA", "DADD", "DMUL",
        "MUFU.RCP64H", "BAR.SYNC", "WARPSYNC", "ACQBULK"]
EXCERPT = {"k_small_coop": ["UBLKCP", "SYNCS", "REDG.E.MIN.64"],
           "k_raster_depth_tiles": ["LDGSTS", "REDG.E.MIN.64"],
           "k_raster_setup": ["ATOMG", "BAR.SYNC"],
           "k_frame_init": ["DFMA"]}

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
funcs = OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    if cur and re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
        funcs[cur].append(line.split(";")[0].strip())


def demangle(name):
    out = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    return out.split("(")[0] if out else name


print(f"SASS audit of {LIB} ({len(funcs)} kernels)\n")
print(f"{'kernel':34s} {'instr':>6s} " + " ".join(f"{k.split('.')[0][:6] if k != 'REDG.E.MIN.64' else 'REDMIN':>6s}"
                                                 for k in KEYS))
rows = []
for f, ins in funcs.items():
    c = Counter()
    for i in ins:
        op = re.sub(r"^/\*[0-9a-f]+\*/\s*", "", i)
        op = re.sub(r"^@!?U?P\w+\s+", "", op)
        for k in KEYS:
            if op.startswith(k):
                c[k] += 1
    c["REDG"] -= c["REDG.E.MIN.64"]
    rows.append((demangle(f), len(ins), c))
for name, n, c in sorted(rows, key=lambda r: -r[1]):
    if not name.startswith("k_") and "k_" not in name:
        continue
    print(f"{name[:34]:34s} {n:6d} " + " ".join(f"{c[k]:6d}" for k in KEYS))

print("\nExcerpts (first occurrence of each opcode, with 2 lines of context):")
for f, ins in funcs.items():
    name = demangle(f)
    for key, ops in EXCERPT.items():
        if name != key and not name.endswith(" " + key) and name.split("<")[0] != key:
            continue
        print(f"\n== {name}")
        for op in ops:
            for j, i in enumerate(ins):
                if re.search(r"\b" + re.escape(op), i):
                    for line in ins[max(0, j - 2): j + 3]:
                        print("   ", line)
                    print("    ...")
                    break
