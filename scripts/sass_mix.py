"""Opcode mix of the hottest loop of a kernel in a cubin/object (run here, no GPU).

usage: python scripts/sass_mix.py <obj> <function-substring> [units_per_iter] [skip_lo:skip_hi ...]
Finds backward branches, takes the loop whose body holds the most FFMA, and
prints its opcode histogram (per loop iteration and per unit if given).
"""
import re, subprocess, sys
from collections import Counter

obj, fsub = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else None
skips = [tuple(int(v, 16) for v in a.split(":")) for a in sys.argv[4:]]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
cands = [f for f in funcs[1:] if fsub in f.split("\n")[0]]
if not cands:
    sys.exit("function not found")
body = cands[0]
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        addr = int(m.group(1), 16)
        txt = m.group(2).strip()
        ins.append((addr, txt))
best = None
import os
if os.environ.get("RANGE"):
    lo, hi = (int(v, 16) for v in os.environ["RANGE"].split(":"))
    seg = [t for a, t in ins if lo <= a <= hi and not any(l2 <= a < h2 for l2, h2 in skips)]
    best = (0, lo, hi, seg)
for i, (addr, txt) in enumerate(ins):
    if best is not None and os.environ.get("RANGE"):
        break
    m = re.search(r"BRA[^;]*?0x([0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt < addr:
        seg = [t for a, t in ins if tgt <= a <= addr and not any(lo <= a < hi for lo, hi in skips)]
        n_ffma = sum(1 for t in seg if re.match(r"(@!?U?P\d\s+)?FFMA", t))
        if best is None or n_ffma > best[0]:
            best = (n_ffma, tgt, addr, seg)
if best is None:
    sys.exit("no loop found")
n_ffma, tgt, addr, seg = best
ops = Counter()
for t in seg:
    t = re.sub(r"^@!?U?P[T\d]+\s+", "", t)
    ops[t.split()[0].split(".")[0]] += 1
tot = sum(ops.values())
print(f"loop {tgt:#x}..{addr:#x}: {tot} instructions")
for a, t in ins:
    if tgt <= a <= addr and ("BRA" in t or "BAR" in t):
        print(f"    {a:#06x} {t}")
for op, c in ops.most_common():
    print(f"  {op:10s} {c:6d}" + (f"  {c/units:6.2f}/unit" if units else ""))
if units:
    print(f"  total/unit {tot/units:.2f}")
