"""Per-kernel totals and shares from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    k = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "").split("(")[0][:60]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
unit = "us" if max(v[1] for v in agg.values()) > 1e4 else "ns"
print(f"{len(rows) - hdr - 1} launches, {tot / 1e3:.1f} us total (gpu__time_duration.sum, serialised, cold)")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{t / 1e3:10.1f} us {n:5d}x {100 * t / tot:5.1f}%  {k}")
