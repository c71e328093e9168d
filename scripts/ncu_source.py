"""Per-region stall attribution from an ncu source page (SASS).

usage: python scripts/ncu_source.py <rep> [chunk] [kernel regex]
Prints chunks of consecutive SASS instructions holding >1% of stall samples,
with their top stall reasons and opcodes.
"""
import csv, io, subprocess, sys
rep = sys.argv[1]
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 64
kf = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *kf, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i]
data = []
for r in rows[i + 1:]:
    if r and r[0] == "Address":
        break  # next kernel's section
    if len(r) == len(h):
        data.append(dict(zip(h, r)))
sc = [k for k in h if k.startswith("stall_")]
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(d[S] or 0) for d in data) or 1
base = int(data[0]["Address"], 16)
print(f"samples {tot}, instructions {len(data)}")
for i in range(0, len(data), chunk):
    seg = data[i:i + chunk]
    s = sum(int(d[S] or 0) for d in seg)
    if s < 0.01 * tot:
        continue
    ex = sum(int(d["Instructions Executed"] or 0) for d in seg)
    agg = {k: sum(int(d[k] or 0) for d in seg) for k in sc}
    top = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:4])
    ops = {}
    for d in seg:
        t = d["Source"].split()
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    topops = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:5])
    a0 = int(seg[0]["Address"], 16) - base
    print(f"{a0:#07x} {100 * s / tot:5.1f}% exec {ex:>10} | {top} | {topops}")
