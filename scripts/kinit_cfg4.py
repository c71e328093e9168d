"""cfg4 k-means++ alone (4M-point 3D map, K=2048): device time per call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
ctx = gm.Context(0)
ctx.upload(p)
for _ in range(reps):
    r = ctx.fit_k_resident(k, gm.EmParams(1, 0.0, 1e-6, 0))
    print(f"kinit {r.ms_kinit:.2f} ms  layout {r.ms_layout:.2f}  m0 {r.ms_mstep0:.2f}  em(1 it) {r.ms_em:.2f}", flush=True)
