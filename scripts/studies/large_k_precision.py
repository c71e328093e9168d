"""End-to-end parameter error vs the FP64 oracle as points per component shrink (large K)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as orc
import paper_2307_00071_b200 as gm
from parity import ll_err, model_err

ctx = gm.Context(0)
frame = gm.synthetic_frame_cloud()
cases = [(16, 512), (8, 1024), (4, 2048), (2, 2048)] if len(sys.argv) < 2 else \
    [tuple(int(v) for v in c.split(":")) for c in sys.argv[1:]]
for stride, k in cases:
    p = frame[::stride].copy()
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    res = gm.fit_k(p, k, em, ctx=ctx, want_labels=True)
    ref = orc.fit_k(p, k, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
    e = model_err(res.model.weights, res.model.means, res.model.covariances,
                  ref["w"], ref["mu"], ref["cov"])
    print(f"n={len(p)} k={k} pts/comp={len(p) / k:.0f} iters {res.em_iterations}/"
          f"{ref['em_iterations']} centres_equal {np.array_equal(res.centers, ref['centers'])} "
          f"ll {ll_err(res.ll_trace, ref['ll_trace']):.2e} err w/mu/cov "
          f"{e[0]:.2e} {e[1]:.2e} {e[2]:.2e}", flush=True)
