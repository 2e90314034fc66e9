"""Per-iteration kernel breakdown of an ncu launch list (--csv,
gpu__time_duration.sum): the launches between two consecutive k_arnoldi
launches, grouped by (kernel, grid).

usage: python tools/iter_breakdown.py launches.csv [iteration index]
"""
import collections
import csv
import io
import sys


def load(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    out = []
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1.0)
        name = r["Kernel Name"].split("(")[0].replace("pmgr::<unnamed>::", "").replace("void ", "").replace("unnamed>::", "")
        out.append((name, r["Grid Size"], v))
    return out


def main(path, which=1):
    L = load(path)
    idx = [i for i, (n, g, v) in enumerate(L) if n.startswith("k_arnoldi")]
    a, b = idx[which], idx[which + 1]
    seg = L[a + 1:b + 1]
    print(f"# launches/iteration {len(seg)}  sum {sum(v for _, _, v in seg):.1f} us")
    agg = collections.OrderedDict()
    for n, g, v in seg:
        agg.setdefault((n, g), [0, 0.0])
        agg[(n, g)][0] += 1
        agg[(n, g)][1] += v
    print("#  total_us    n   avg_us  kernel")
    for (n, g), (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:45]:
        print(f"  {t:9.1f} {c:3d} {t / c:8.1f}  {n} grid={g}")
    small = sum(t for (c, t) in agg.values() if t / c < 60)
    ns = sum(c for (c, t) in agg.values() if t / c < 60)
    print(f"# kernels under 60 us: {ns} launches, {small:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
