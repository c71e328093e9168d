"""BASELINE configurations at their stated sizes (marked slow: the FP64
oracle needs minutes here).

cfg4: the 4M-point 3D map (make_structured_scene x 25 + (100, -40, 0) m),
K=2048, k-means++ + EM to tol 1e-3 — unsharded and as 8 virtual ranks
(the point-sharded path of SURVEY.md §8(e)). cfg5's largest K: the cfg2
frame with K=4096. The oracle side is kinit (sogmm.cpp:197-337) + the
hard M step (:481, m_step on one-hot log_gamma) + the streaming EM loop
(:484-509 without the N x K matrix, bit-identical to the materialised one),
which is fit(cloud, K) with K given.
"""
import numpy as np
import pytest

from parity import LL_TOL, assert_model_close, ll_err

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def oracle_fit_k_streaming(orc, p, k, tol, seed=0, max_iters=100):
    lab, cen = orc.kinit(p, k, seed)
    w, mu, cov, removed = orc.m_step_labels(p, lab, k, 1e-6)
    d = p.shape[1]
    ref = orc.fit_from(p, w, mu[:, :d].copy(), cov[:, :d * (d + 1) // 2].copy(),
                       max_iters=max_iters, ll_rel_tol=tol, cov_reg=1e-6, streaming=True)
    return lab, cen, removed, ref


def check_fit(res, lab, cen, removed, ref, labels=None):
    assert np.array_equal(res.centers, cen)
    assert np.array_equal(res.labels if labels is None else labels, lab)
    assert res.em_iterations == ref["em_iterations"]
    assert res.removed_components == removed + ref["removed"]
    assert ll_err(res.ll_trace, ref["ll_trace"]) < LL_TOL
    m = res.model
    return assert_model_close(m.weights, m.means, m.covariances, ref["w"], ref["mu"], ref["cov"])


def test_cfg4_full_size_unsharded_and_vshard8(gm, orc, ctx):
    p = gm.structured_scene(4_000_000, 4, 0.005)[:, :3] * 25 + np.array([100.0, -40.0, 0.0])
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    res = gm.fit_k(p, 2048, em, ctx=ctx, want_labels=True)
    rs = gm.fit_k_vsharded(p, 2048, em, world=8, want_labels=True)
    lab, cen, removed, ref = oracle_fit_k_streaming(orc, p, 2048, 1e-3)
    errs = check_fit(res, lab, cen, removed, ref)
    errs8 = check_fit(rs[0], lab, cen, removed, ref,
                      labels=np.concatenate([r.labels for r in rs]))
    print("cfg4 errors (w, mu, cov): 1 GPU", errs, "8 virtual ranks", errs8)


# FP64 self-sensitivity of this trajectory (profiles/r2_em_sensitivity.txt,
# scripts/studies/em_sensitivity_k4096.py): perturbing the reference's own
# initial means by a relative 1e-7 (FP32 rounding) moves its final
# parameters by (2.1e-4, 1.7e-4, 1.5e-3) after the 11 EM iterations (~15,000x
# amplification at ~75 points per component); 1e-9 moves them by 1.5e-5.
# The 1e-4 end-to-end parameter bar is therefore below the reference's own
# noise floor here; the kernel is held to 1e-5 per step (teacher-forced) and
# the trajectory to the integer / ll bars plus that floor.
K4096_E2E_FLOOR = 1.5e-3


def test_cfg5_k4096_end_to_end(gm, orc, ctx):
    p = gm.synthetic_frame_cloud()
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    res = gm.fit_k(p, 4096, em, ctx=ctx, want_labels=True)
    lab, cen, removed, ref = oracle_fit_k_streaming(orc, p, 4096, 1e-3)
    assert np.array_equal(res.centers, cen)
    assert np.array_equal(res.labels, lab)
    assert res.em_iterations == ref["em_iterations"]
    assert res.removed_components == removed + ref["removed"]
    assert ll_err(res.ll_trace, ref["ll_trace"]) < LL_TOL
    m = res.model
    errs = assert_model_close(m.weights, m.means, m.covariances, ref["w"], ref["mu"], ref["cov"],
                              tol=K4096_E2E_FLOOR)
    # teacher-forced: one E + M step from the oracle's model after 5 iterations
    w, mu, cov, _ = orc.m_step_labels(p, lab, 4096, 1e-6)
    mid = orc.fit_from(p, w, mu, cov, max_iters=5, ll_rel_tol=0.0, cov_reg=1e-6, streaming=True)
    one = gm.fit_from(p, gm.Gmm(mid["w"], mid["mu"], mid["cov"]), gm.EmParams(1, 0.0, 1e-6),
                      ctx=ctx)
    r1 = orc.fit_from(p, mid["w"], mid["mu"], mid["cov"], max_iters=1, ll_rel_tol=0.0,
                      cov_reg=1e-6, streaming=True)
    assert abs(one.final_log_likelihood - r1["final_ll"]) / abs(r1["final_ll"]) < LL_TOL
    step = assert_model_close(one.model.weights, one.model.means, one.model.covariances,
                              r1["w"], r1["mu"], r1["cov"], tol=1e-5)
    print("cfg5 K=4096 end-to-end errors (w, mu, cov):", errs, "per step:", step,
          "iterations", res.em_iterations)
