"""Summarise an ncu --csv launch list (gpu__time_duration.sum and optional
dram bytes) per kernel: total time, share, launches, average, DRAM GB/s.

usage: python tools/launch_summary.py launches.csv [header lines...]
"""

import csv
import io
import sys
from collections import defaultdict


def main(path, header=()):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = defaultdict(dict)
    for r in rows:
        per[r["ID"]]["name"] = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        else:
            v *= {"Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1.0)
        per[r["ID"]][r["Metric Name"]] = v
    agg = defaultdict(lambda: [0.0, 0, 0.0])
    for d in per.values():
        name = d["name"].split("(")[0].replace("pmgr::<unnamed>::", "").replace("void ", "")
        a = agg[name]
        a[0] += d.get("gpu__time_duration.sum", 0.0)
        a[1] += 1
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(a[0] for a in agg.values())
    out = list(header)
    out.append(f"# launches={len(per)}  sum of kernel times={total / 1e3:.2f} ms")
    out.append("# total_us   share  launches  avg_us  dram_GB/s  kernel")
    for name, (t, n, b) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        gbs = b / (t * 1e-6) / 1e9 if t > 0 else 0.0
        out.append(f"{t:10.0f} {100 * t / total:6.1f}% {n:9d} {t / n:7.2f} {gbs:10.0f}  {name}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
