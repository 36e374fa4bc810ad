"""Instruction mix of one kernel from an ncu report's SASS source page:
    ncu -i rep --page source --csv --kernel-name regex:NAME --print-source sass > x.csv
    python tools/sass_mix.py x.csv [units]    (units: divide counts, e.g. work items)"""
import csv
import sys
from collections import Counter

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 6 and r[0].startswith("0x")]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ops, tot = Counter(), 0
for r in rows:
    n = int(r[5] or 0)
    tot += n
    toks = r[1].strip().split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    ops[op.split(".")[0]] += n
print(f"total {tot}  per unit {tot / units:.1f}")
for op, n in ops.most_common(32):
    print(f"{op:10s} {n:12d} {n / units:9.1f}")
