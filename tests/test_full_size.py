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


def test_cfg5_k4096_end_to_end(gm, orc, ctx):
    p = gm.synthetic_frame_cloud()
    em = gm.EmParams(100, 1e-3, 1e-6, 0)
    res = gm.fit_k(p, 4096, em, ctx=ctx, want_labels=True)
    lab, cen, removed, ref = oracle_fit_k_streaming(orc, p, 4096, 1e-3)
    errs = check_fit(res, lab, cen, removed, ref)
    print("cfg5 K=4096 errors (w, mu, cov):", errs, "iterations", res.em_iterations)
