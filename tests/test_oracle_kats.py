"""Pins the FP64 oracle (oracle/oracle.cpp) against the known-answer tests
SPEC.md states for the hot path (the reference ships no tests or golden
vectors: proj/tests/CMakeLists.txt is empty). CPU only.

SPEC.md anchors: cholesky_cache :81-83, batched_cholesky :189-191,
logsumexp_rows :207-211/:225, weighted_moments :219-221, kinit :283-285,
e_step :293-296, m_step :304-306, fit :314-322, acceptance 2-3 :648-649.
"""
import math

import numpy as np
import pytest


LN2PI = math.log(2 * math.pi)


def spd(rng, m, d=4, eps=1e-3):
    a = rng.normal(size=(m, d, d))
    return np.einsum("mij,mkj->mik", a, a) + eps * np.eye(d)


def pack(s):
    r, c = np.tril_indices(s.shape[-1])
    # packed10 order is row-major lower: (0,0),(1,0),(1,1),(2,0)...
    order = sorted(zip(r, c))
    idx = tuple(np.array(x) for x in zip(*order))
    return s[..., idx[0], idx[1]]


# ---- cholesky_cache / batched_cholesky --------
def test_cholesky_identity(orc):
    lo, pr, ld = orc.cholesky_cache(pack(np.eye(4))[None])
    assert np.array_equal(lo[0], np.eye(4))
    assert np.array_equal(pr[0], np.eye(4))
    assert ld[0] == 0.0


def test_cholesky_diag(orc):
    lo, pr, ld = orc.cholesky_cache(pack(np.diag([4.0, 1, 1, 1]))[None])
    assert np.array_equal(lo[0], np.diag([2.0, 1, 1, 1]))
    assert abs(ld[0] - math.log(0.5)) < 1e-15  # -0.693147


@pytest.mark.parametrize("m", [100, 1000])
def test_cholesky_random_reconstruct(orc, m):
    rng = np.random.default_rng(m)
    s = spd(rng, m)
    lo, pr, ld = orc.cholesky_cache(pack(s))
    assert np.max(np.abs(lo @ lo.transpose(0, 2, 1) - s)) < 1e-10
    assert np.allclose(np.triu(lo, 1), 0.0)
    # log_det_terms = -1/2 ln|Sigma| (SPEC invariant, within 1e-8)
    assert np.max(np.abs(-2 * ld - np.linalg.slogdet(s)[1])) < 1e-8
    assert np.max(np.abs(pr @ lo - np.eye(4))) < 1e-10


def test_cholesky_non_spd_reports_first_block(orc):
    s = np.stack([np.eye(4), np.eye(4), -np.eye(4), -np.eye(4)])
    with pytest.raises(orc.OracleError) as e:
        orc.cholesky_cache(pack(s))
    assert e.value.code == 3 and "block 2" in str(e.value)


# ---- logsumexp_rows -----------------------------
def test_logsumexp_kats(orc):
    ninf = -np.inf
    m = np.array([[0.0, 0.0, ninf], [1000.0, ninf, ninf], [ninf, ninf, ninf]])
    out = orc.logsumexp_rows(m)
    assert abs(out[0] - math.log(2)) < 1e-15
    assert out[1] == 1000.0
    assert out[2] == ninf


def test_logsumexp_random_and_shift(orc):
    rng = np.random.default_rng(1)
    m = rng.normal(size=(100, 50)) * 3
    out = orc.logsumexp_rows(m)
    naive = np.log(np.exp(m).sum(axis=1))
    assert np.max(np.abs(out - naive) / np.abs(naive)) < 1e-12
    out2 = orc.logsumexp_rows(m + 123.25)
    assert np.max(np.abs(out2 - (out + 123.25))) < 1e-12


# ---- weighted_moments ----------------------------------
def test_weighted_moments_uniform(orc):
    rng = np.random.default_rng(2)
    x = rng.normal(size=(5000, 4))
    counts, means, sc, deg = orc.weighted_moments(x, np.ones((5000, 1)))
    assert abs(counts[0] - 5000) < 1e-9
    assert np.allclose(means[0], x.mean(0), rtol=0, atol=1e-12)
    assert np.allclose(sc[0], np.cov(x.T, bias=True), rtol=0, atol=1e-12)


def test_weighted_moments_indicator_and_naive(orc):
    rng = np.random.default_rng(3)
    x = rng.normal(size=(3000, 4))
    lab = rng.integers(0, 3, 3000)
    resp = np.eye(3)[lab]
    counts, means, sc, deg = orc.weighted_moments(x, resp)
    for b in range(3):
        xs = x[lab == b]
        assert counts[b] == len(xs)
        assert np.allclose(means[b], xs.mean(0), atol=1e-12)
        assert np.allclose(sc[b], np.cov(xs.T, bias=True), atol=1e-12)
    # random responsibilities vs a naive loop
    r = rng.random((3000, 5))
    r /= r.sum(1, keepdims=True)
    counts, means, sc, deg = orc.weighted_moments(x, r)
    for b in range(5):
        w = r[:, b]
        mu = (w[:, None] * x).sum(0) / w.sum()
        d = x - mu
        s = (w[:, None, None] * d[:, :, None] * d[:, None, :]).sum(0) / w.sum()
        assert np.allclose(means[b], mu, atol=1e-10)
        assert np.allclose(sc[b], s, atol=1e-10)


# ---- kinit ----------------------------------------------
def blobs(gm, per=200, sigma=0.01, seed=5):
    c = np.array([[0.1, 0.1, 0.1, 0.1], [0.5, 0.5, 0.5, 0.5], [0.9, 0.9, 0.9, 0.9]])
    return gm.blob_cloud(c, sigma, per, seed), c


def test_kinit_k1(orc, gm):
    x, _ = blobs(gm)
    lab, cen = orc.kinit(x, 1, 0)
    assert np.all(lab == 0)


def test_kinit_k_equals_n_is_permutation(orc):
    rng = np.random.default_rng(4)
    x = np.column_stack([rng.normal(size=(50, 3)), rng.random(50)])
    lab, cen = orc.kinit(x, 50, 0)
    assert sorted(lab.tolist()) == list(range(50))
    assert sorted(cen.tolist()) == list(range(50))


def test_kinit_three_blobs_partition(orc, gm):
    x, c = blobs(gm)
    lab, cen = orc.kinit(x, 3, 0)
    truth = np.repeat(np.arange(3), 200)
    # partition equality up to label permutation
    for b in range(3):
        assert len(set(lab[truth == b].tolist())) == 1
    assert len(set(lab.tolist())) == 3


def test_kinit_every_component_owns_a_point_with_duplicates(orc):
    # 40 copies of 5 distinct points: k = 8 > distinct => fallback + fix-up
    base = np.array([[0, 0, 0, 0.1], [1, 0, 0, 0.2], [0, 1, 0, 0.3], [0, 0, 1, 0.4],
                     [1, 1, 1, 0.5]], float)
    x = np.repeat(base, 40, axis=0)
    lab, cen = orc.kinit(x, 8, 0)
    assert np.all(np.bincount(lab, minlength=8) >= 1)


def test_kinit_invalid_k(orc, gm):
    x, _ = blobs(gm, per=5)
    with pytest.raises(orc.OracleError) as e:
        orc.kinit(x, 16, 0)
    assert e.value.code == 2


# ---- e_step --------------------------------------------
def test_estep_single_component(orc, gm):
    x, _ = blobs(gm)
    lg, ll = orc.e_step(x, [1.0], [[0.5] * 4], pack(np.eye(4) * 0.1)[None])
    assert np.max(np.abs(lg)) < 1e-12


def test_estep_identical_components(orc, gm):
    x, _ = blobs(gm)
    cov = pack(np.eye(4) * 0.1)
    lg, ll = orc.e_step(x, [0.5, 0.5], [[0.5] * 4] * 2, np.stack([cov, cov]))
    assert np.max(np.abs(np.exp(lg) - 0.5)) < 1e-12


def test_estep_standard_normal_density(orc):
    lg, ll = orc.e_step(np.zeros((1, 4)), [1.0], [[0.0] * 4], pack(np.eye(4))[None])
    assert abs(ll - (-2 * LN2PI)) < 1e-12  # -3.675754


def test_estep_matches_linear_domain_and_direct_density(orc):
    """Eq. (3) equivalence (acceptance 2): Cholesky form = direct inverse/det."""
    rng = np.random.default_rng(6)
    s = spd(rng, 3, eps=0.5)
    mu = rng.normal(size=(3, 4))
    w = np.array([0.2, 0.3, 0.5])
    x = np.column_stack([rng.normal(size=(200, 3)), rng.random(200)])
    lg, ll = orc.e_step(x, w, mu, pack(s))
    dens = np.zeros((200, 3))
    for b in range(3):
        d = x - mu[b]
        q = np.einsum("ni,ij,nj->n", d, np.linalg.inv(s[b]), d)
        dens[:, b] = math.log(w[b]) - 0.5 * (4 * LN2PI + q + np.linalg.slogdet(s[b])[1])
    lse = np.log(np.exp(dens).sum(1))
    assert abs(ll - lse.sum()) / abs(lse.sum()) < 1e-10
    assert np.max(np.abs(lg - (dens - lse[:, None]))) < 1e-8
    # rows logsumexp to 0 within 1e-9
    assert np.max(np.abs(np.log(np.exp(lg).sum(1)))) < 1e-9


# ---- m_step ---------------------------------------------
def test_mstep_uniform_mle(orc):
    rng = np.random.default_rng(7)
    x = np.column_stack([rng.normal(size=(4000, 3)), rng.random(4000)])
    w, mu, cov, rm = orc.m_step(x, np.zeros((4000, 1)), 1e-6)
    assert rm == 0 and w[0] == 1.0
    assert np.allclose(mu[0], x.mean(0), atol=1e-12)
    assert np.allclose(cov[0], pack(np.cov(x.T, bias=True) + 1e-6 * np.eye(4)), atol=1e-12)


def test_mstep_degenerate_removed_and_renumbered(orc):
    rng = np.random.default_rng(8)
    x = np.column_stack([rng.normal(size=(1000, 3)), rng.random(1000)])
    lg = np.full((1000, 3), -np.inf)
    lg[:500, 0] = 0.0
    lg[500:, 2] = 0.0
    w, mu, cov, rm = orc.m_step(x, lg, 1e-6)
    assert rm == 1 and len(w) == 2
    assert np.allclose(mu[1], x[500:].mean(0), atol=1e-12)
    lg[:] = -np.inf
    with pytest.raises(orc.OracleError) as e:
        orc.m_step(x, lg, 1e-6)
    assert "all components degenerate" in str(e.value)


def test_mstep_labels_equals_onehot_mstep(orc, gm):
    x, _ = blobs(gm)
    lab, cen = orc.kinit(x, 5, 0)
    lg = np.full((len(x), 5), -np.inf)
    lg[np.arange(len(x)), lab] = 0.0
    a = orc.m_step(x, lg, 1e-6)
    b = orc.m_step_labels(x, lab, 5, 1e-6)
    for u, v in zip(a[:3], b[:3]):
        assert np.array_equal(u, v)


# ---- fit / EM (acceptance 3) -----------------------------
def test_em_monotone_rows_and_blob_recovery(orc, gm):
    hits = 0
    for seed in range(10):
        x, c = blobs(gm, per=300, sigma=0.02, seed=100 + seed)
        r = orc.fit_k(x, 3, max_iters=50, ll_rel_tol=1e-10, cov_reg=1e-6, seed=seed)
        tr = r["ll_trace"]
        assert np.all(np.diff(tr) >= -1e-8 * np.abs(tr[:-1]))
        lg, _ = orc.e_step(x, r["w"], r["mu"], r["cov"])
        assert np.max(np.abs(np.log(np.exp(lg).sum(1)))) < 1e-9
        tol = 3 * 0.02 / math.sqrt(300)
        d = np.abs(np.sort(r["mu"][:, 0]) - c[:, 0])
        hits += bool(np.all(d < tol))
    assert hits >= 9


def test_fit_deterministic_and_thread_independent(orc, gm):
    x, _ = blobs(gm, per=400, seed=9)
    orc.set_num_threads(1)
    a = orc.fit_k(x, 6, max_iters=30, ll_rel_tol=1e-9)
    orc.set_num_threads(8)
    b = orc.fit_k(x, 6, max_iters=30, ll_rel_tol=1e-9)
    orc.set_num_threads(0)
    for k in ("w", "mu", "cov", "ll_trace"):
        assert np.array_equal(a[k], b[k]), k


def test_fit_streaming_matches_materialised(orc, gm):
    x, _ = blobs(gm, per=500, seed=10)
    lab, cen = orc.kinit(x, 4, 0)
    w, mu, cov, _ = orc.m_step_labels(x, lab, 4, 1e-6)
    a = orc.fit_from(x, w, mu, cov, max_iters=10, ll_rel_tol=0.0)
    b = orc.fit_from(x, w, mu, cov, max_iters=10, ll_rel_tol=0.0, streaming=True)
    assert a["em_iterations"] == b["em_iterations"] == 10
    assert np.max(np.abs(a["ll_trace"] - b["ll_trace"]) / np.abs(a["ll_trace"])) < 1e-12
    assert np.max(np.abs(a["mu"] - b["mu"])) < 1e-12


def test_em_loop_returns_model_semantics(orc, gm):
    """sogmm.cpp:488-509: max-iters exit returns the model one M step past
    the last ll; the tolerance exit returns the model that produced it."""
    x, _ = blobs(gm, per=300, seed=11)
    lab, cen = orc.kinit(x, 3, 0)
    w, mu, cov, _ = orc.m_step_labels(x, lab, 3, 1e-6)
    one = orc.fit_from(x, w, mu, cov, max_iters=1, ll_rel_tol=0.0)
    lg, ll = orc.e_step(x, w, mu, cov)
    w2, mu2, cov2, _ = orc.m_step(x, lg, 1e-6)
    assert one["final_ll"] == ll and np.array_equal(one["mu"], mu2)
    conv = orc.fit_from(x, w, mu, cov, max_iters=200, ll_rel_tol=1e-3)
    assert conv["em_iterations"] < 200
    lg3, ll3 = orc.e_step(x, conv["w"], conv["mu"], conv["cov"])
    assert ll3 == conv["final_ll"]


def test_validation_errors(orc):
    x = np.zeros((10, 4))
    x[3, 1] = np.nan
    with pytest.raises(orc.OracleError) as e:
        orc.kinit(x, 2, 0)
    assert e.value.code == 3
    x = np.zeros((10, 4))
    x[2, 3] = 1.5
    with pytest.raises(orc.OracleError) as e:
        orc.kinit(x, 2, 0)
    assert "intensity" in str(e.value)


def test_3d_embedding_constant(orc, gm):
    """3D clouds run as [x,y,z,0]: ll_4D - ll_3D = N(-1/2 ln 2pi - 1/2 ln reg)."""
    x = gm.structured_scene(3000, 2, 0.005)[:, :3]
    r3 = orc.fit_k(x, 8, max_iters=5, ll_rel_tol=0.0, cov_reg=1e-6)
    x4 = np.column_stack([x, np.zeros(len(x))])
    r4 = orc.fit_k(x4, 8, max_iters=5, ll_rel_tol=0.0, cov_reg=1e-6)
    off = orc.ll_offset_3d(len(x), 1e-6)
    assert np.max(np.abs(r4["ll_trace"] - off - r3["ll_trace"]) / np.abs(r3["ll_trace"])) < 1e-12
    assert np.array_equal(r3["mu"], r4["mu"][:, :3])
