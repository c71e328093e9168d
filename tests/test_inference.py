"""§8(f) inference rows: score, joint_dist_sample, color_conditional and
the dense e_step API, CUDA path (C ABI) vs the FP64 oracle restatement of
inference.cpp / sogmm.cpp on identical inputs.

Bars: FP64 arithmetic on both sides with different log/exp/sin/cos
implementations (CUDA vs glibc) and summation orders -> 1e-10 relative on
scores and draws; sampled component choices exact (integer)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def model(gm, orc):
    p = gm.synthetic_frame_cloud()[::7]
    r = orc.fit_k(p, 48, 60, 1e-4, 1e-6, 2)
    return p, r["w"], r["mu"], r["cov"]


def test_score_matches_oracle(gm, orc, ctx, model):
    p, w, mu, cov = model
    avg, pp = gm.score(p, gm.Gmm(w, mu, cov), ctx=ctx, per_point=True)
    ref = orc.score(p, w, mu, cov)
    assert abs(avg - ref) <= 1e-10 * abs(ref)
    assert abs(pp.mean() - ref) <= 1e-10 * abs(ref)


def test_e_step_api_matches_oracle(gm, orc, ctx, model):
    p, w, mu, cov = model
    lg, ll = gm.e_step(p, gm.Gmm(w, mu, cov), ctx=ctx)
    rlg, rll = orc.e_step(p, w, mu, cov)
    assert abs(ll - rll) <= 1e-10 * abs(rll)
    ok = rlg > -700
    assert np.max(np.abs(lg[ok] - rlg[ok])) <= 1e-8


def test_sample_matches_oracle(gm, orc, ctx, model):
    _, w, mu, cov = model
    n = 20000
    x = gm.joint_dist_sample(gm.Gmm(w, mu, cov), n, 11, ctx=ctx)
    rx = orc.sample(w, mu, cov, n, 11)
    scale = np.maximum(np.abs(rx), 1.0)
    assert np.max(np.abs(x - rx) / scale) <= 1e-10
    # determinism and counter independence: draw i depends only on (seed, i)
    x2 = gm.joint_dist_sample(gm.Gmm(w, mu, cov), 100, 11, ctx=ctx)
    assert np.array_equal(x2, x[:100])


def test_sample_moments(gm, ctx):
    w = np.array([0.3, 0.7])
    mu = np.array([[0.0, 0.0, 0.0, 0.2], [1.0, 2.0, 3.0, 0.8]])
    cov = np.array([[0.04, 0.0, 0.04, 0.0, 0.0, 0.04, 0.0, 0.0, 0.0, 0.01],
                    [0.09, 0.02, 0.09, 0.0, 0.0, 0.09, 0.0, 0.0, 0.0, 0.01]])
    x = gm.joint_dist_sample(gm.Gmm(w, mu, cov), 400000, 5, ctx=ctx)
    mean = w @ mu
    assert np.allclose(x.mean(axis=0), mean, atol=5e-3)


def test_sample_3d(gm, ctx):
    w = np.array([1.0])
    mu = np.array([[1.0, -2.0, 0.5]])
    cov = np.array([[0.25, 0.1, 0.25, 0.0, 0.0, 0.01]])
    x = gm.joint_dist_sample(gm.Gmm(w, mu, cov), 200000, 1, ctx=ctx)
    assert x.shape == (200000, 3)
    assert np.allclose(x.mean(axis=0), mu[0], atol=5e-3)
    c = np.cov(x.T)
    assert abs(c[0, 1] - 0.1) < 5e-3 and abs(c[2, 2] - 0.01) < 1e-3


@pytest.mark.parametrize("clamp", [True, False])
def test_color_conditional_matches_oracle(gm, orc, ctx, model, clamp):
    p, w, mu, cov = model
    locs = np.vstack([p[:3000, :3], p[:50, :3] + 40.0])  # + far queries (underflow fallback)
    e, v = gm.color_conditional(gm.Gmm(w, mu, cov), locs, clamp, ctx=ctx)
    re_, rv = orc.color_conditional(w, mu, cov, locs, clamp)
    assert np.max(np.abs(e - re_)) <= 1e-9
    assert np.max(np.abs(v - rv)) <= 1e-9 * max(1.0, float(np.max(rv)))
    assert np.all(v >= 0)


def test_inference_errors(gm, ctx):
    w = np.array([0.5, 0.5])
    mu = np.zeros((2, 4))
    bad = np.array([[1, 0, 1, 0, 0, 1, 0, 0, 0, 1], [1, 2, 1, 0, 0, 1, 0, 0, 0, 1]], float)
    with pytest.raises(gm.NumericalError, match="component 1 is not positive definite"):
        gm.score(np.zeros((4, 4)) + 0.5, gm.Gmm(w, mu, bad), ctx=ctx)
    with pytest.raises(gm.NumericalError, match="weights sum"):
        gm.joint_dist_sample(gm.Gmm(np.array([0.5, 0.6]), mu, bad), 10, ctx=ctx)
    with pytest.raises(ValueError):
        gm.joint_dist_sample(gm.Gmm(w, mu, bad), 0, ctx=ctx)
