"""Top SASS lines by warp-stall samples from an ncu --page source --csv dump.
python tools/src_top.py one_x.src.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Source" in r)
h = rows[hdr]
j = h.index("Warp Stall Sampling (All Samples)")
k = h.index("Warp Stall Sampling (Not-issued Samples)")
data = rows[hdr + 1:]


def val(r, c):
    try:
        return float(r[c])
    except (ValueError, IndexError):
        return 0.0


tot = sum(val(r, j) for r in data)
print(f"total samples {tot:.0f}")
for r in sorted(data, key=lambda r: -val(r, j))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{val(r, j):6.0f} {val(r, k):6.0f}  {r[0][-5:]}  {r[1][:90]}")
