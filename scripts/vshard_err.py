"""tests/test_vshard.py frame case: fit errors vs the FP64 oracle for the
unsharded and the 2-rank virtual-shard fit, dense and pruned E steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as orc
import paper_2307_00071_b200 as gm
from parity import model_err, ll_err

p = gm.synthetic_frame_cloud()[::2].copy()
k = 128
em = gm.EmParams(100, 1e-3, 1e-6, 0)
ref = orc.fit_k(p, k, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, seed=0)
for mode in ("dense", "pruned"):
    os.environ["GMMB_ESTEP"] = "dense" if mode == "dense" else "sparse"
    ctx = gm.Context(0)
    one = gm.fit_k(p, k, em, ctx=ctx)
    for world in (1, 2, 4):
        r = one if world == 1 else gm.fit_k_vsharded(p, k, em, world=world)[0]
        e = model_err(r.model.weights, r.model.means, r.model.covariances, ref["w"], ref["mu"], ref["cov"])
        print(f"{mode} world={world} iters {r.em_iterations}/{ref['em_iterations']} "
              f"ll {ll_err(r.ll_trace, ref['ll_trace']):.2e} w {e[0]:.2e} mu {e[1]:.2e} cov {e[2]:.2e}",
              flush=True)
    ctx.close()
