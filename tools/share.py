"""Per-category shares of an ncu launch list (python tools/share.py launches.csv steps)."""
import re
import sys
from collections import defaultdict

import csv


def load(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out = []
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            out.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) *
                        scale.get(r["Metric Unit"], 1.0)))
    return out


CATS = [("radius/CSR/CSC", r"k_radius|k_stable_bucket|k_scan|k_histogram|k_csc|k_csr|k_count|k_fill_idx|k_place"),
        ("agg fwd", r"k_agg_fwd"), ("agg bwd", r"k_agg_bwd"),
        ("force edges", r"k_force_"), ("EGNN edge / tanh / head", r"k_egnn"),
        ("tcgen05 GEMM", r"tc_gemm"),
        ("split-K / colsum", r"splitk|colsum"), ("loss / Adam / guard", r"k_loss|k_adam|k_nonfinite|k_sgd"),
        ("other", r".")]
rows = load(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot = sum(t for _, t in rows)
acc = defaultdict(float)
for name, t in rows:
    for c, pat in CATS:
        if re.search(pat, name):
            acc[c] += t
            break
for c, _ in CATS:
    print(f"{c:20s} {acc[c] / steps:9.1f} us/step  {100 * acc[c] / tot:5.1f}%")
print(f"{'total':20s} {tot / steps:9.1f} us/step")
print()
print("# top kernels (us summed over the step)")
print(f"launches: {len(rows) // steps}")
by = defaultdict(lambda: [0.0, 0])
for name, t in rows:
    k = name[:100]
    by[k][0] += t
    by[k][1] += 1
for k, (t, n) in sorted(by.items(), key=lambda x: -x[1][0])[:20]:
    print(f"{t / steps:9.1f} us  {n // steps:4d}x {k}")
