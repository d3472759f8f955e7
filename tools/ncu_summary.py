"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel.
Usage: python tools/ncu_summary.py launches.csv [n_steps]"""
import collections
import csv
import re
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")[:70]
    v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches "
      f"({tot / steps:.1f} us per step for {steps:g} steps)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}% {v[0]:5d}x  {k}")
