"""One cfg4 fit (4M-point 3D map, K = 2048) on the resident cloud (ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
ctx = gm.Context(0)
if os.environ.get("GMMB_TIMING", "0") == "1":
    ctx.set_timing(True)
s = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
ctx.upload(s)
r = ctx.fit_k_resident(2048, gm.EmParams(int(os.environ.get("ITERS", "3")), 0.0, 1e-6, 0))
print(r.em_iterations, r.ms_kinit, r.ms_em, r.ms_total)
