"""Blackwell-native evidence from the shipped library: per kernel, counts of the SASS
instructions that prove tcgen05 / TMEM / TMA use (B200_PROFILING.md table) -- UTC*MMA
(tcgen05.mma), UTCBAR (tcgen05.commit), LDTM / STTM (tcgen05.ld / st), UTMALDG / UTMASTG
(TMA tensor load / store), UBLKCP (bulk copy) -- and HMMA (the legacy mma.sync path).

    python tools/sass_counts.py [lib] > profiles/round2_sass_counts.md
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2306_09342_b200/_lib/librevprop_b200.so"
OPS = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP",
       "UTMAPF", "HMMA", "MUFU.EX2"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
counts = defaultdict(Counter)
func = None
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        func = m.group(1)
        continue
    if func is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    for o in OPS:
        if op == o or op.startswith(o + "."):
            counts[func][o] += 1


def pretty(f):
    try:
        return subprocess.run(["c++filt"], input=f, capture_output=True, text=True).stdout.strip()[:110]
    except Exception:
        return f[:110]


print(f"# SASS evidence per kernel ({LIB}, cuobjdump -sass; static instruction counts)\n")
print("| kernel | " + " | ".join(OPS) + " |")
print("|---|" + "---|" * len(OPS))
for f in sorted(counts, key=lambda x: pretty(x)):
    c = counts[f]
    if not any(c[o] for o in OPS):
        continue
    print(f"| `{pretty(f)}` | " + " | ".join(str(c[o]) for o in OPS) + " |")
