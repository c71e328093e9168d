"""Debug: with a -DGMMB_SP_COUNT build (GMMB_LIB) and GMMB_DEBUG=1, the
driver prints per EM run the tasks taken by the pruned E kernel (units x
iterations + the split sub-units when nothing is taken twice)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2307_00071_b200 as gm
k = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = gm.Context(0)
if len(sys.argv) > 2 and sys.argv[2] == "cfg4":
    p = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
else:
    p = gm.synthetic_frame_cloud()
ctx.upload(p)
for it in (1, 2, 3, 5, 8):
    r = ctx.fit_k_resident(k, gm.EmParams(it, 0.0, 1e-6, 0))
    print("iters", r.em_iterations, flush=True)
