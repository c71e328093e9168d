"""How much does the FP64 reference trajectory itself move under a tiny
perturbation at cfg5 K=4096 (the cfg2 frame, ~75 points per component)?

Runs the oracle (kinit -> hard M step -> streaming EM to tol 1e-3) twice:
once as is, once with the initial model perturbed by a relative 1e-9 (far
below FP32 rounding). The final-parameter difference, in the parity metrics
of tests/parity.py, is the floor any implementation that is not bitwise
identical to the reference can reach on this configuration.
"""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np
import oracle
from parity import model_err, ll_err

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-9
p = oracle.synthetic_frame_cloud()
t = time.time()
lab, cen = oracle.kinit(p, k, 0)
w, mu, cov, _ = oracle.m_step_labels(p, lab, k, 1e-6)
print("kinit + M0", round(time.time() - t, 1), "s", flush=True)
a = oracle.fit_from(p, w, mu, cov, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, streaming=True)
rng = np.random.default_rng(0)
mu2 = mu * (1 + eps * rng.standard_normal(mu.shape))
b = oracle.fit_from(p, w, mu2, cov, max_iters=100, ll_rel_tol=1e-3, cov_reg=1e-6, streaming=True)
print("iterations", a["em_iterations"], b["em_iterations"])
print("ll trace rel diff", ll_err(b["ll_trace"], a["ll_trace"]))
print("final (w, mu, cov) diff for a %g relative perturbation of the initial means:" % eps,
      model_err(b["w"], b["mu"], b["cov"], a["w"], a["mu"], a["cov"]))
