"""Per-kernel share of a ncu --metrics gpu__time_duration.sum launch list."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'us':>10} {'launches':>8} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:10.1f} {v[0]:8d} {100 * v[1] / tot:5.1f}%  {k}")
print(f"{tot:10.1f} total (cold-cache, serialised by ncu: compare shares)")
