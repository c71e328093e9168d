"""One cfg4-size kinit (for ncu) + the tile kernel's exchange count."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
s = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
ctx = gm.Context(0)
for _ in range(int(os.environ.get("REPS", "1"))):
    lab, cen = gm.kinit(s, 2048, 0, ctx=ctx)
print("ok", cen[:4])
