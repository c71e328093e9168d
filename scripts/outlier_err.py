"""Teacher-forced EM steps: parameter errors vs the FP64 oracle for the dense
E step, the pruned one, and the pruned kernel with every pair kept
(GMMB_SPARSE_QCUT=1e30, set per process: run this file with --keep-all).
Cases: the far-outlier test of tests/test_gpu_parity.py and plain scenes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as orc
import paper_2307_00071_b200 as gm
from parity import model_err
from test_gpu_parity import fixed_init

tag = "keepall" if os.environ.get("GMMB_SPARSE_QCUT") else "pruned"
for k, seed, far_on in [(64, 9, True), (1024, 9, True), (64, 3, False), (64, 4, False),
                        (256, 5, False), (512, 6, False)]:
    base = gm.structured_scene(30000, seed, 0.005)
    w, mu, cov = fixed_init(orc, base, k)
    p = base
    if far_on:
        far = base[:40].copy()
        far[:, :3] += 3.0
        p = np.vstack([base, far])
    lg, rll = orc.e_step(p, w, mu, cov)
    rw, rmu, rcov, rrm = orc.m_step(p, lg, 1e-6)
    for dense in ((True, False) if tag == "pruned" else (False,)):
        ctx = gm.Context(0)
        ctx.set_estep_mode(dense)
        ll, m1, rm = gm.em_step(p, gm.Gmm(w, mu, cov), 1e-6, ctx=ctx)
        e = model_err(m1.weights, m1.means, m1.covariances, rw, rmu, rcov)
        print(f"k={k} seed={seed} far={far_on} {'dense' if dense else tag}: ll {abs(ll - rll) / abs(rll):.2e} "
              f"w {e[0]:.2e} mu {e[1]:.2e} cov {e[2]:.2e}", flush=True)
        ctx.close()
