"""Per-kernel DRAM traffic of one eager RevViT-B Reprop step, from an ncu CSV of
dram__bytes_read.sum, dram__bytes_write.sum and gpu__time_duration.sum, aggregated per
kernel kind; writes the GEMM traffic file bench.py reports as roofline.traffic.

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,\\
        gpu__time_duration.sum --clock-control none --csv --log-file traffic.csv \\
        python tools/profile_step.py --mode reprop
    python tools/gemm_traffic.py traffic.csv profiles/round2_gemm_traffic
"""
import csv
import json
import re
import sys
from collections import defaultdict


def kind(name):
    m = re.search(r"gemm_sm100(_2sm)?_kernel<(.*?)>", name)
    if m:
        return "gemm<" + m.group(2).replace(" ", "") + ">"
    return re.sub(r"\(.*", "", name).replace("void ", "")[:60]


def main():
    path, out = sys.argv[1], sys.argv[2]
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    per = defaultdict(dict)  # launch id -> metrics
    names = {}
    for r in csv.DictReader(lines):
        lid = r["ID"]
        names[lid] = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if r["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            per[lid][r["Metric Name"]] = v * scale
        elif r["Metric Name"] == "gpu__time_duration.sum":
            scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9}.get(unit, 1e-9)
            per[lid]["t"] = v * scale
    agg = defaultdict(lambda: {"launches": 0, "dram_read": 0.0, "dram_write": 0.0, "seconds": 0.0})
    for lid, m in per.items():
        k = kind(names[lid])
        a = agg[k]
        a["launches"] += 1
        a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
        a["seconds"] += m.get("t", 0.0)
    gemm = [a for k, a in agg.items() if k.startswith("gemm")]
    n = sum(a["launches"] for a in gemm)
    tot = sum(a["dram_read"] + a["dram_write"] for a in gemm)
    res = {"source": path, "kinds": agg, "gemm_launches": n,
           "avg_dram_bytes_per_launch": tot / max(n, 1)}
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    T = sum(a["seconds"] for a in agg.values())
    rows = ["| kernel kind | launches | ms | share | DRAM read MB/launch | DRAM write MB/launch | "
            "achieved GB/s |", "|---|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["seconds"]):
        L = a["launches"]
        rows.append(f"| {k} | {L} | {a['seconds'] * 1e3:.3f} | {100 * a['seconds'] / T:.1f}% | "
                    f"{a['dram_read'] / L / 1e6:.1f} | {a['dram_write'] / L / 1e6:.1f} | "
                    f"{(a['dram_read'] + a['dram_write']) / max(a['seconds'], 1e-12) / 1e9:.0f} |")
    with open(out + ".md", "w") as f:
        f.write(f"# DRAM traffic per kernel kind, one eager RevViT-B Reprop step (B = 256), ncu "
                f"(serialised, cold caches)\n\ntotal {T * 1e3:.3f} ms over "
                f"{sum(a['launches'] for a in agg.values())} launches; GEMM average "
                f"{res['avg_dram_bytes_per_launch'] / 1e6:.1f} MB per launch over {n} launches\n\n")
        f.write("\n".join(rows) + "\n")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
