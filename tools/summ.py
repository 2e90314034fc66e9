"""One-line summaries of bench JSON files: ms/step, iterations, per-kernel us and GB/s."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    c = d.get("config", {})
    print(f, f"{d.get('value', 0):.3f} {d.get('unit')}", f"{d.get('ms_per_step', 0):.2f} ms",
          "its", c.get("gmres_iterations"), "setup", round(d.get("setup_s") or 0, 3),
          "e2e", round((d.get("e2e") or {}).get("ms_per_step") or 0, 2))
    for k, v in (d.get("kernels") or {}).items():
        print("   ", k, round(v["avg_us"] or 0, 2), "us", round(v["gbs"] or 0), "GB/s")
