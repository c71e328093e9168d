"""Decode SASS control words (stall count, yield, barriers) of a range and
estimate single-warp issue cycles (B300_MICROARCH.md control-word layout).

usage: python scripts/sass_ctrl.py <sass-dump> lo hi [--print]
<sass-dump>: output of `cuobjdump -sass` restricted to one function.
"""
import re, sys
path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
show = "--print" in sys.argv
lines = open(path).read().split("\n")
ins = []
for i, line in enumerate(lines):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", line)
    if not m:
        continue
    a = int(m.group(1), 16)
    m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
    hiw = int(m2.group(1), 16)
    ctrl = hiw >> 41
    stall = ctrl & 0xF
    yld = (ctrl >> 4) & 1
    wbar = (ctrl >> 5) & 7
    rbar = (ctrl >> 8) & 7
    wait = (ctrl >> 11) & 0x3F
    if lo <= a <= hi:
        ins.append((a, m.group(2).strip(), stall, yld, wbar, rbar, wait))
tot = sum(x[2] for x in ins)
from collections import Counter
c = Counter()
for a, t, s, y, wb, rb, w in ins:
    op = re.sub(r"^@!?U?P[T\d]+\s+", "", t).split()[0].split(".")[0]
    c[(op, s)] += 1
    if show:
        print(f"{a:#06x} s={s:2d} y={y} wb={wb} rb={rb} w={w:06b} {t}")
print(f"{len(ins)} instructions, sum of stall counts {tot} (cycles/warp lower bound ignoring SB waits)")
for (op, s), n in sorted(c.items(), key=lambda x: -x[1] * x[0][1])[:15]:
    print(f"  {op:8s} stall={s:2d} x{n}")
