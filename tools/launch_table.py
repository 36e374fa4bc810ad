"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_table.py gpurun_out/launches.csv [--md]
"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name) if "gemm" not in name else name
    m = re.search(r"gemm_sm100\w*<(.*)>", name)
    if m:
        return "gemm<" + m.group(1)[:60] + ">"
    return name[:70]


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v
        rows.append((short(r["Kernel Name"]), ms))
    agg = defaultdict(lambda: [0, 0.0])
    for k, ms in rows:
        agg[k][0] += 1
        agg[k][1] += ms
    tot = sum(ms for _, ms in rows)
    print(f"total {tot:.3f} ms over {len(rows)} launches\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")


if __name__ == "__main__":
    main()
