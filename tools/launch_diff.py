"""Per-kernel time difference of two ncu launch lists (same workload):
python tools/launch_diff.py a.csv b.csv"""
import csv
import re
import sys
from collections import defaultdict


def load(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    acc = defaultdict(float)
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            name = re.sub(r"\(.*", "", r["Kernel Name"])[:90]
            acc[name] += float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1.0)
    return acc


a, b = load(sys.argv[1]), load(sys.argv[2])
rows = sorted(set(a) | set(b), key=lambda k: -abs(a.get(k, 0) - b.get(k, 0)))
print(f"{'kernel':90s} {'A us':>9s} {'B us':>9s} {'A-B':>8s}")
for k in rows[:25]:
    print(f"{k:90s} {a.get(k, 0):9.1f} {b.get(k, 0):9.1f} {a.get(k, 0) - b.get(k, 0):8.1f}")
print(f"{'total':90s} {sum(a.values()):9.1f} {sum(b.values()):9.1f}")
