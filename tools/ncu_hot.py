"""Top SASS lines of an ncu source page (csv) by warp-stall samples, with the
stall reasons that dominate each.   ncu -i X.ncu-rep --page source --csv
--print-source sass > f.csv ; python tools/ncu_hot.py f.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_") or "Stall" in x and i != si]
tot = sum(float(r[si] or 0) for r in data)
print(f"total samples {tot:.0f}")
idx = sorted(range(len(data)), key=lambda i: -float(data[i][si] or 0))[:n]
for i in sorted(idx):
    r = data[i]
    print(f"{i:5d} {float(r[si]):7.0f} {100 * float(r[si]) / tot:5.1f}%  {r[1].strip()[:80]}")
